#!/bin/bash
# The reference package's full config-3-shaped Newton solve at 96^3 (2.7M DOF) on the box's
# host cores (extends the measured ladder 16^3-64^3), and the live composition at the same size.
set -u
mkdir -p gpurun_out
timeout 2700 python tools/cpu_reference.py ladder 96 > gpurun_out/r02_cpu_ladder96.jsonl 2> gpurun_out/r02_cpu_ladder96.err
echo "ladder rc=$?"
timeout 600 python -c "
import sys, json; sys.path.insert(0, 'tools'); import cpu_reference as cr
c = cr.ReferenceComposer(n_target=96, n_csr=64)
print(json.dumps({'composer_96': c.step()}))" > gpurun_out/r02_composer96.json 2>&1
echo "composer rc=$?"
cut -c1-600 gpurun_out/r02_cpu_ladder96.jsonl; cut -c1-400 gpurun_out/r02_composer96.json
