#!/bin/bash
# GRID3 with the self block packed to its 6 upper entries (this build) against the previous
# build's 9-entry self block (libb200fem_prev.so swapped in): GPU suite, iteration profile, solve.
# (The packed layout was reverted after this measurement: no gain, profiles/r02_selfpack_ab.jsonl.)
set -u
mkdir -p gpurun_out
L=paper_2212_00964_b200
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/sp_gputests.log 2>&1; echo "gputests rc=$?"; tail -2 gpurun_out/sp_gputests.log
cp $L/libb200fem.so /tmp/libnew.so
for i in 1 2; do
  for v in new prev; do
    if [ $v = prev ]; then cp $L/libb200fem_prev.so $L/libb200fem.so; else cp /tmp/libnew.so $L/libb200fem.so; fi
    python tools/krylov_profile.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['lib']='$v'; print(json.dumps(d))" >> gpurun_out/r02_selfpack_ab.jsonl
  done
done
for v in new prev; do
  if [ $v = prev ]; then cp $L/libb200fem_prev.so $L/libb200fem.so; else cp /tmp/libnew.so $L/libb200fem.so; fi
  timeout 900 python tools/newton_ab.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['lib']='$v'; print(json.dumps(d))" >> gpurun_out/r02_selfpack_ab.jsonl
done
cp /tmp/libnew.so $L/libb200fem.so
B200FEM_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_spmv_grid3' -c 6 --csv --log-file gpurun_out/r02_selfpack_ncu.csv python tools/ncu_targets.py spmv > /dev/null 2>&1
echo "ncu rc=$?"
cat gpurun_out/r02_selfpack_ab.jsonl | cut -c1-330
