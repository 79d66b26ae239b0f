timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/c31_gputests.log 2>&1; echo "gputests rc=$?"; tail -3 gpurun_out/c31_gputests.log
for v in 0 1; do
  if [ $v = 1 ]; then export B200FEM_GRID_PF_NORMAL=1; else unset B200FEM_GRID_PF_NORMAL; fi
  B200FEM_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:'k_spmv_grid3' -c 8 --csv --log-file gpurun_out/r02_jacobi_modes_ncu_$v.csv \
      python tools/ncu_targets.py spmv > /dev/null 2>&1
  echo "ncu normal=$v rc=$?"
done
