#!/bin/bash
# k_update_xr in one full wave (occupancy-sized grid) vs kRedBlocks = 8 blocks/SM (A/B), and the
# DRAM bytes of the Jacobi-mode matvecs with / without the evict-first operand policy.
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for v in "" 1184; do
    if [ -z "$v" ]; then unset B200FEM_XR_BLOCKS; else export B200FEM_XR_BLOCKS=$v; fi
    python tools/krylov_profile.py 2>/dev/null | tail -1 >> gpurun_out/r02_xr_wave_ab.jsonl
  done
done
unset B200FEM_XR_BLOCKS
timeout 900 python tools/newton_ab.py B200FEM_XR_BLOCKS=1184 >> gpurun_out/r02_xr_wave_ab.jsonl 2>/dev/null
cat gpurun_out/r02_xr_wave_ab.jsonl | cut -c1-330
for v in 0 1; do
  if [ $v = 1 ]; then export B200FEM_GRID_PF_NORMAL=1; else unset B200FEM_GRID_PF_NORMAL; fi
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:'k_spmv_grid3' -c 8 --csv --log-file gpurun_out/r02_jacobi_modes_ncu_$v.csv \
      python tools/ncu_targets.py spmv > /dev/null 2>&1
  echo "ncu normal=$v rc=$?"
done
