#!/bin/bash
# GRID3 matvecs with the first NPF upper value blocks staged through shared memory by cp.async
# (The NPF variants were removed after this measurement: slower, profiles/r02_npf_ab.jsonl.)
# (B200FEM_GRID_NPF = 2 | 4 | 5) against register loads only (A/B).
set -u
mkdir -p gpurun_out
for i in 1 2; do
  for v in 0 2 4 5; do
    B200FEM_GRID_NPF=$v python tools/krylov_profile.py 2>/dev/null | tail -1 >> gpurun_out/r02_npf_ab.jsonl
  done
done
cat gpurun_out/r02_npf_ab.jsonl | cut -c1-300
timeout 1200 python tools/newton_ab.py B200FEM_GRID_NPF=2 B200FEM_GRID_NPF=4 B200FEM_GRID_NPF=5 >> gpurun_out/r02_npf_ab.jsonl 2>gpurun_out/r02_npf_ab.err
tail -4 gpurun_out/r02_npf_ab.jsonl | cut -c1-420
