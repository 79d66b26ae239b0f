"""Diagnostic: in-stream kernel timeline of BiCGSTAB iterations (CUPTI via torch.profiler).

Unlike an ncu launch list (serialised, caches flushed) this shows the kernels as they run
back to back in the solve, including the idle gaps between them.  Diagnostic only; bench
numbers never come from a profiled run.

    python tools/timeline_probe.py [--n 136] [--iters 40] [--method bicgstab|pcg]
"""

import argparse
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import torch  # noqa: E402

import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402
from spmv_probe import problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=136)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--method", default="bicgstab")
    ap.add_argument("--material", default="nh")
    ap.add_argument("--operator", default="grid", choices=["csr", "grid"], help="grid: the Newton operator")
    a = ap.parse_args()
    prob = problem(a.n, a.material)
    ws = fem.workspace(prob)
    N = prob.n_dofs
    U = D.zeros(N)
    K = fem.solvers._tangent_matrix(prob, U, a.operator)
    R = D.empty(N)
    ws.residual(prob, U, R)
    b = -R
    cfg = fem.LinearSolveConfig(rel_tol=1e-300, abs_tol=1e-300, max_iters=a.iters, method=a.method)

    def run():
        try:
            fem.solvers._bicgstab_device(K, b, D.zeros(N), False, cfg)
        except fem.LinearSolverError:
            pass
        torch.cuda.synchronize()

    run()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    per = collections.defaultdict(list)
    gaps = collections.defaultdict(list)
    prev = None
    for e in ev:
        name = e.name.split("(")[0].replace("void ", "").replace("b200::", "")[:48]
        dur = e.time_range.end - e.time_range.start
        if prev is not None and dur > 5.0:  # launches after convergence exit in ~2 us: skip them
            gaps[name].append(e.time_range.start - prev.time_range.end)
        if dur > 5.0:
            per[name].append(dur)
        prev = e
    span = ev[-1].time_range.end - ev[0].time_range.start
    out = {"span_us": span, "n_kernels": len(ev), "kernels": {}}
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        g = gaps.get(k, [0])
        q = max(1, len(v) // 10)
        out["kernels"][k] = {"n": len(v), "avg_us": sum(v) / len(v), "first10pct_us": sum(v[:q]) / q,
                             "last10pct_us": sum(v[-q:]) / q, "tot_us": sum(v),
                             "gap_before_avg_us": sum(g) / max(1, len(g))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
