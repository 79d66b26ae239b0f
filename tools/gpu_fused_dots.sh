#!/bin/bash
# Two-allreduce partitioned BiCGSTAB (B200FEM_DIST_FUSED_DOTS): dist tests, then the 8-part
# local-mode config-3 solve and the 1-rank NCCL bench with the fused dot group off and on.
set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/fused_tests.log 2>&1; echo "dist tests rc=$?"
tail -3 gpurun_out/fused_tests.log
for f in 0 1; do
  B200FEM_DIST_FUSED_DOTS=$f timeout 600 python tools/dist_local_check.py --parts 8 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['fused_dots']=$f; print(json.dumps(d))" \
    >> gpurun_out/r02_dist_fused_ab.jsonl
done
for f in 0 1; do
  B200FEM_DIST_FUSED_DOTS=$f timeout 600 python bench.py --spawn --steps 3 --warmup 3 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'fused_dots': $f, 'value': d['value'], 'linear_iterations': d['newton']['linear_iterations'], 'in_solve_iter_ms': d['newton']['in_solve_iter_ms'], 'parallelism': d['config']['parallelism']}))" \
    >> gpurun_out/r02_dist_fused_ab.jsonl
done
cat gpurun_out/r02_dist_fused_ab.jsonl | cut -c1-600
bash tools/gpu_ncu_hot.sh > gpurun_out/r02b_ncu.log 2>&1; echo "ncu rc=$?"
