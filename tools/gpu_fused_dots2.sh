#!/bin/bash
# Two-allreduce partitioned BiCGSTAB after moving its scratch allocation out of the graph
# capture: dist + grid tests, 8-part local solve and 1-rank NCCL bench with the fused dot group off / on.
# Run after the capture fix (private capture stream, scratch allocated before capture).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_grid.py -x -q > gpurun_out/fd2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/fd2_tests.log
for f in 0 1; do
  B200FEM_KRYLOV_TRACE=1 B200FEM_DIST_FUSED_DOTS=$f timeout 600 python tools/dist_local_check.py --parts 8 2> gpurun_out/fd2_local_$f.err \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['fused_dots']=$f; d['mode']='local 8 parts'; print(json.dumps(d))" >> gpurun_out/r02_dist_fused_ab2.jsonl
  grep -m1 "batch graph" gpurun_out/fd2_local_$f.err
done
for f in 0 1; do
  B200FEM_DIST_FUSED_DOTS=$f timeout 600 python bench.py --spawn --partitioned --steps 3 --warmup 3 --no-alt --no-cpu-baseline 2>/dev/null | grep '^{' | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'fused_dots': $f, 'mode': '1-rank NCCL (bench --spawn --partitioned)', 'value': d['value'], 'linear_iterations': d['newton']['linear_iterations'], 'parallelism': d['config']['parallelism']}))" \
    >> gpurun_out/r02_dist_fused_ab2.jsonl
done
cut -c1-300 gpurun_out/r02_dist_fused_ab2.jsonl
