#!/bin/bash
# Evict-first L2 policy on the prefetched row operands of the Jacobi-mode GRID3 matvecs (A/B),
# and the partitioned path through a 1-rank NCCL communicator with 3 vs 2 allreduces.
set -u
mkdir -p gpurun_out
timeout 900 python tools/newton_ab.py B200FEM_GRID_PF_NORMAL=1 > gpurun_out/r02_pf_policy_ab.jsonl 2> gpurun_out/r02_pf_policy_ab.err
cat gpurun_out/r02_pf_policy_ab.jsonl | cut -c1-700
for v in 0 1; do
  if [ $v = 1 ]; then export B200FEM_GRID_PF_NORMAL=1; else unset B200FEM_GRID_PF_NORMAL; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:'k_spmv_grid3' -c 4 --csv --log-file gpurun_out/r02_pf_policy_ncu_$v.csv \
      python tools/ncu_targets.py spmv > /dev/null 2>&1
  echo "ncu policy normal=$v rc=$?"
done
unset B200FEM_GRID_PF_NORMAL
for f in 0 1; do
  B200FEM_DIST_FUSED_DOTS=$f timeout 600 python bench.py --spawn --partitioned --steps 3 --warmup 3 2>/dev/null | tail -1 \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'fused_dots': $f, 'value': d['value'], 'linear_iterations': d['newton']['linear_iterations'], 'in_solve_iter_ms': d['newton']['in_solve_iter_ms'], 'parallelism': d['config']['parallelism']}))" \
    >> gpurun_out/r02_dist_fused_ab.jsonl
done
tail -2 gpurun_out/r02_dist_fused_ab.jsonl
