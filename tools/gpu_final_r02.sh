#!/bin/bash
# End-of-round evidence on one B200: GPU test suite, smoke(), the default bench line, the
# reference arm, the 1-rank partitioned bench through the spawn path, and the bench command's
# kernel launch list.  Outputs in gpurun_out/ (f_*).
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/f_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q > $O/f_gputests.log 2>&1; echo "gputests rc=$?" >> $O/f_status.txt
tail -3 $O/f_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/f_smoke.log 2>&1; echo "smoke rc=$?" >> $O/f_status.txt
timeout 900 python bench.py > $O/f_bench.json 2> $O/f_bench.err; echo "bench rc=$?" >> $O/f_status.txt
timeout 900 python bench.py --impl reference > $O/f_bench_ref.json 2> $O/f_bench_ref.err; echo "bench ref rc=$?" >> $O/f_status.txt
timeout 900 python bench.py --spawn --partitioned --steps 3 --warmup 3 --no-alt --no-cpu-baseline > $O/f_bench_spawn1.json 2> $O/f_bench_spawn1.err; echo "spawn rc=$?" >> $O/f_status.txt
B200FEM_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/f_launches.csv python bench.py --steps 1 --warmup 0 --no-alt --no-cpu-baseline > $O/f_ncu_bench.log 2>&1; echo "ncu rc=$?" >> $O/f_status.txt
cat $O/f_status.txt
