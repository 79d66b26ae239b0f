"""Diagnostic: burst vs sustained (power-capped) bandwidth of a plain copy and of the SpMV.

Runs each workload back to back for --seconds, timing every launch with CUDA events, and
samples nvidia-smi (SM clock, power, event reasons) in the background.  Prints one JSON
line per workload: first-launch-window and last-window GB/s, and the clock/power medians
seen while it ran.

    python tools/power_probe.py [--n 136] [--seconds 4]
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2212_00964_b200 as fem  # noqa: E402
from paper_2212_00964_b200 import _device as D  # noqa: E402
from paper_2212_00964_b200 import _lib  # noqa: E402
from spmv_probe import problem  # noqa: E402


class Smi:
    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = "clocks.sm,power.draw,clocks_event_reasons.active"
        while not self._stop.is_set():
            try:
                o = subprocess.run(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=5).stdout.strip().split(",")
                self.samples.append((time.perf_counter(), float(o[0]), float(o[1]), o[2].strip()))
            except Exception:
                pass
            time.sleep(0.1)

    def window(self, t0, t1):
        s = [x for x in self.samples if t0 <= x[0] <= t1]
        if not s:
            return {}
        return {"sm_mhz_median": float(np.median([x[1] for x in s])), "power_w_median": float(np.median([x[2] for x in s])),
                "reasons": sorted(set(x[3] for x in s))}

    def stop(self):
        self._stop.set()
        self._t.join()


def sustained(fn, nbytes, seconds):
    evs = []
    t0 = time.perf_counter()
    torch.cuda.synchronize()
    while time.perf_counter() - t0 < seconds:
        batch = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            batch.append((a, b))
        torch.cuda.synchronize()
        evs += [a.elapsed_time(b) / 1e3 for a, b in batch]
    t1 = time.perf_counter()
    k = max(1, len(evs) // 10)
    return {"launches": len(evs), "burst_gbs": nbytes / np.mean(evs[:k]) / 1e9,
            "sustained_gbs": nbytes / np.mean(evs[-3 * k:]) / 1e9, "last_us": float(np.mean(evs[-3 * k:]) * 1e6),
            "first_us": float(np.mean(evs[:k]) * 1e6)}, t0, t1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=136)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--no-copy", action="store_true")
    a = ap.parse_args()
    smi = Smi()
    time.sleep(0.5)
    if not a.no_copy:
        copy_probe(smi, a.seconds)
    spmv_probe(smi, a)
    smi.stop()


def copy_probe(smi, seconds):
    src = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
    dst = torch.empty_like(src)
    src.fill_(1)
    res, t0, t1 = sustained(lambda: dst.copy_(src), 2 * src.numel() * 2, seconds)
    print(json.dumps({"workload": "torch copy 2 GiB (read+write)", **res, **smi.window(t0, t1)}), flush=True)
    del src, dst
    time.sleep(2.0)


def spmv_probe(smi, a):
    prob = problem(a.n, "nh")
    ws = fem.workspace(prob)
    N = prob.n_dofs
    K = fem.assemble_jacobian(prob, D.zeros(N))
    x = D.to_device(np.random.default_rng(0).standard_normal(N))
    y = D.empty(N)
    lib, h = _lib.lib(), K._device_handle()
    nnz, nn = ws.nnz, prob.mesh.n_nodes
    nbytes = 8 * nnz + 4 * (nnz // 9) + 4 * (nn + 1) + 16 * N
    time.sleep(2.0)
    res, t0, t1 = sustained(lambda: lib.b200fem_matvec(h, D.ptr(x), D.ptr(y)), nbytes, a.seconds)
    print(json.dumps({"workload": "SpMV config 3 (plain)", "x_variant": os.environ.get("B200FEM_SPMV_X", "scalar"),
                      **res, **smi.window(t0, t1)}), flush=True)


if __name__ == "__main__":
    main()
