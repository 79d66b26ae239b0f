set -x
for n in 136 160 200; do
  timeout 300 python tools/spmv_probe.py --operator grid --n $n --reps 20 --iters 2 > gpurun_out/probe_$n.log 2>&1
  B200FEM_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_spmv_grid3 -c 3 --csv python tools/spmv_probe.py --operator grid --n $n --reps 3 --iters 2 > gpurun_out/ncu_size_$n.csv 2>gpurun_out/ncu_size_$n.err
done
