#!/bin/bash
# r02 bench evidence: the default bench line, the 1-rank partitioned solve through the spawn path,
# and the launch list of the bench command (ncu, host batch loop so the Krylov kernels are visible).
cd "$(dirname "$0")/.."
O=gpurun_out
python bench.py > $O/c9_bench.json 2> $O/c9_bench.err; echo "bench rc=$?" >> $O/c9_status.txt
python bench.py --spawn --partitioned --steps 3 --warmup 3 --no-alt --no-cpu-baseline > $O/c9_bench_spawn1.json 2> $O/c9_bench_spawn1.err; echo "spawn rc=$?" >> $O/c9_status.txt
B200FEM_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/c9_launches.csv python bench.py --steps 1 --warmup 0 --no-alt --no-cpu-baseline > $O/c9_ncu_bench.log 2>&1; echo "ncu rc=$?" >> $O/c9_status.txt
cat $O/c9_status.txt
