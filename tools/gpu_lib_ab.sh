#!/bin/bash
# Library A/B by swapping a variant build (paper_2212_00964_b200/libb200fem_$1.so) in for the
# default one: NH tangent and residual time at config 3 (tools/spmv_probe.py), 3 rounds each.
set -u
V=$1
L=paper_2212_00964_b200
mkdir -p gpurun_out
cp $L/libb200fem.so /tmp/lib_base.so
for i in 1 2 3; do
  for v in base $V; do
    if [ $v = base ]; then cp /tmp/lib_base.so $L/libb200fem.so; else cp $L/libb200fem_$V.so $L/libb200fem.so; fi
    python tools/spmv_probe.py --operator grid --n 136 --reps 5 --iters 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$v', 'jacobian_ms': d['jacobian_ms'], 'residual_ms': d['residual_ms'], 'spmv_us': d['spmv_us']}))" >> gpurun_out/r02_lib_ab_$V.jsonl
  done
done
cp /tmp/lib_base.so $L/libb200fem.so
cat gpurun_out/r02_lib_ab_$V.jsonl
