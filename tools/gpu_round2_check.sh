#!/bin/bash
# One GPU-box pass: full GPU test suite, tangent-kernel A/B and the fused kernel under the
# parity tests, the bench line (ours + reference arm), composer validation.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/c2_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/c2_gputests.log 2>&1; echo "gputests rc=$?" >> $O/c2_status.txt
timeout 600 python tools/tangent_ab.py --n 136 > $O/c2_tangent_ab.jsonl 2> $O/c2_tangent_ab.err; echo "tangent_ab rc=$?" >> $O/c2_status.txt
B200FEM_TANGENT=fused timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_parity.py tests/test_gpu_nhcube.py tests/test_gpu_dist.py tests/test_gpu_grid_slab.py -x -q > $O/c2_fused_tests.log 2>&1; echo "fused tests rc=$?" >> $O/c2_status.txt
timeout 900 python bench.py --steps 3 --warmup 3 > $O/c2_bench.json 2> $O/c2_bench.err; echo "bench rc=$?" >> $O/c2_status.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/c2_bench_ref.json 2> $O/c2_bench_ref.err; echo "bench ref rc=$?" >> $O/c2_status.txt
timeout 600 python -c "
import sys, json; sys.path.insert(0, 'tools'); import cpu_reference as cr
c = cr.ReferenceComposer(n_target=64, n_csr=64)
print(json.dumps({'composer_64': c.step(), 'ladder_64_measured_total_s': 451.1}))" > $O/c2_composer64.json 2>&1; echo "composer rc=$?" >> $O/c2_status.txt
cat $O/c2_status.txt
