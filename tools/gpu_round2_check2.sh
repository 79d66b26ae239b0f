#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/c3_gputests.log 2>&1; echo "gputests rc=$?" >> $O/c3_status.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/c3_bench.json 2> $O/c3_bench.err; echo "bench rc=$?" >> $O/c3_status.txt
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_cases.py > $O/c3_memcheck.log 2>&1; echo "memcheck rc=$?" >> $O/c3_status.txt
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > $O/c3_racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/c3_status.txt
cat $O/c3_status.txt
