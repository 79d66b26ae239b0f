for cfg in "16 128" "8 128" "16 600"; do
  set -- $cfg
  env B200FEM_PAIR=1 B200FEM_NO_GRAPH=1 B200FEM_GRID_SLAB=$1 B200FEM_PAIR_LAG=$2 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio,smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__inst_executed.sum --clock-control none -k regex:k_grid3_pair -c 1 --csv python tools/spmv_probe.py --operator grid --n 136 --reps 1 --iters 2 > gpurun_out/pair_m_$1_$2.csv 2>&1
done
