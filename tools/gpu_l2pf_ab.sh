#!/bin/bash
# GRID3 matvecs with the upper value tiles of the work item 1 / 2 waves ahead bulk-prefetched
# (The L2PF variant was removed after this measurement: slower, profiles/r02_l2pf_ab.jsonl.)
# into L2 (B200FEM_GRID_L2PF) against no prefetch (A/B).
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for v in 0 1 2; do
    B200FEM_GRID_L2PF=$v python tools/krylov_profile.py 2>/dev/null | tail -1 >> gpurun_out/r02_l2pf_ab.jsonl
  done
done
cat gpurun_out/r02_l2pf_ab.jsonl | cut -c1-300
for v in 0 1; do
  B200FEM_GRID_L2PF=$v python tools/spmv_probe.py --operator grid --n 136 --reps 20 --iters 20 2>&1 | tail -1 | sed "s/^/l2pf=$v /"
done
