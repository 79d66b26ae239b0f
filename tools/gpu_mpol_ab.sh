#!/bin/bash
# L2 eviction priority of the matrix values (and x) in the Jacobi-mode GRID3 matvecs (A/B).
# The B200FEM_GRID_MPOL variants were removed after this measurement (profiles/r02_mpol_ab.jsonl).
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for v in 0 1 2; do
    B200FEM_GRID_MPOL=$v python tools/krylov_profile.py 2>/dev/null | tail -1 >> gpurun_out/r02_mpol_ab.jsonl
  done
done
cat gpurun_out/r02_mpol_ab.jsonl | cut -c1-300
for v in 1 2; do
  B200FEM_GRID_MPOL=$v B200FEM_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:'k_spmv_grid3' -c 6 --csv --log-file gpurun_out/r02_mpol_ncu_$v.csv \
      python tools/ncu_targets.py spmv > /dev/null 2>&1
  echo "ncu mpol=$v rc=$?"
done
