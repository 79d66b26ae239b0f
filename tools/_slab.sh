timeout 600 python -m pytest tests/test_gpu_grid.py tests/test_gpu_dist.py -x -q -m gpu > gpurun_out/slab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/slab_tests.log
for sl in 0 -1 8 16 48; do
  for n in 136 160 200; do
    if [ $sl = -1 ]; then unset B200FEM_GRID_SLAB; else export B200FEM_GRID_SLAB=$sl; fi
    echo "slab=$sl $(timeout 300 python tools/spmv_probe.py --operator grid --n $n --reps 20 --iters 20 2>&1 | tail -1)"
  done
done > gpurun_out/slab_sweep.log
unset B200FEM_GRID_SLAB
for n in 160 200; do
B200FEM_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_spmv_grid3 -c 2 --csv python tools/spmv_probe.py --operator grid --n $n --reps 2 --iters 2 > gpurun_out/ncu_slab_$n.csv 2>gpurun_out/ncu_slab_$n.err
done
