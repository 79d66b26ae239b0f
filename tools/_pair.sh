# A/B of the matvec-pair BiCGSTAB iteration: "pair slab_rows lag_margin" (slab -1 = auto)
timeout 600 python -m pytest tests/test_gpu_pair.py -x -q > gpurun_out/pair_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/pair_tests.log
for cfg in "0 -1 128" "1 -1 128" "1 16 128" "1 16 400" "1 8 128"; do
  set -- $cfg
  for n in 136; do
    echo "pair=$1 slab=$2 lag=$3 $(env B200FEM_PAIR=$1 B200FEM_GRID_SLAB=$2 B200FEM_PAIR_LAG=$3 timeout 300 python tools/spmv_probe.py --operator grid --n $n --reps 3 --iters 30 2>&1 | tail -1)"
  done
done > gpurun_out/pair_probe.log
env B200FEM_PAIR=1 B200FEM_NO_GRAPH=1 B200FEM_GRID_SLAB=16 B200FEM_PAIR_LAG=128 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__inst_executed.sum --clock-control none -k regex:k_grid3_pair -c 1 --csv python tools/spmv_probe.py --operator grid --n 136 --reps 1 --iters 2 > gpurun_out/pair_m2.csv 2>&1
