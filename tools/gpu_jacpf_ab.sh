#!/bin/bash
# Tangent phase A with the next batch's node data prefetched into registers (the default since
# this measurement) against B200FEM_JAC_NO_PF=1: tangent time at config 3, and the GPU suite.
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in 0 1; do
    if [ $v = 1 ]; then unset B200FEM_JAC_NO_PF; else export B200FEM_JAC_NO_PF=1; fi
    python tools/spmv_probe.py --operator grid --n 136 --reps 5 --iters 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'jac_pf': $v, 'jacobian_ms': d['jacobian_ms'], 'residual_ms': d['residual_ms']}))" >> gpurun_out/r02_jacpf_ab.jsonl
  done
done
cat gpurun_out/r02_jacpf_ab.jsonl
unset B200FEM_JAC_NO_PF; timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/jacpf_tests.log 2>&1; echo "tests(pf) rc=$?"; tail -2 gpurun_out/jacpf_tests.log
