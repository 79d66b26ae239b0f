#!/bin/bash
# Library A/B of the BiCGSTAB iteration: this build against a variant build swapped in
# (paper_2212_00964_b200/libb200fem_$1.so), tools/krylov_profile.py alternated 3 times, then
# one Newton solve each (tools/newton_ab.py, baseline only).
set -u
V=$1
L=paper_2212_00964_b200
mkdir -p gpurun_out
cp $L/libb200fem.so /tmp/lib_base.so
for i in 1 2 3; do
  for v in base $V; do
    if [ $v = base ]; then cp /tmp/lib_base.so $L/libb200fem.so; else cp $L/libb200fem_$V.so $L/libb200fem.so; fi
    python tools/krylov_profile.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['lib']='$v'; print(json.dumps(d))" >> gpurun_out/r02_lib_ab_krylov_$V.jsonl
  done
done
for v in base $V; do
  if [ $v = base ]; then cp /tmp/lib_base.so $L/libb200fem.so; else cp $L/libb200fem_$V.so $L/libb200fem.so; fi
  timeout 900 python tools/newton_ab.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); d['lib']='$v'; print(json.dumps(d))" >> gpurun_out/r02_lib_ab_krylov_$V.jsonl
done
cp /tmp/lib_base.so $L/libb200fem.so
cut -c1-330 gpurun_out/r02_lib_ab_krylov_$V.jsonl
