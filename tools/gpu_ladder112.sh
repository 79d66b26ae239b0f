#!/bin/bash
# The reference package's full config-3-shaped Newton solve at 112^3 (4.3M DOF) on the box's
# host cores (extends the measured ladder 16^3-64^3), and the live composition at the same size.
set -u
mkdir -p gpurun_out
timeout 3300 python tools/cpu_reference.py ladder 112 > gpurun_out/r02_cpu_ladder112.jsonl 2> gpurun_out/r02_cpu_ladder112.err
echo "ladder rc=$?"
timeout 600 python -c "
import sys, json; sys.path.insert(0, 'tools'); import cpu_reference as cr
c = cr.ReferenceComposer(n_target=112, n_csr=64)
print(json.dumps({'composer_112': c.step()}))" > gpurun_out/r02_composer112.json 2>&1
echo "composer rc=$?"
cut -c1-600 gpurun_out/r02_cpu_ladder112.jsonl; cut -c1-400 gpurun_out/r02_composer112.json
