"""Probe: device MMA update on n design variables (with asymptote history), timed with CUDA
events; ncu-friendly (python tools/mma_probe.py [--n 340736] [--steps 4])."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2212_00964_b200 import _device as D  # noqa: E402
from paper_2212_00964_b200.inverse import MmaState, mma_update  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=340736)
    ap.add_argument("--steps", type=int, default=4)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    n = a.n
    x = D.to_device(rng.uniform(0.2, 0.9, n))
    c = D.to_device(np.full(n, 1.0 / n))
    st = MmaState.fresh(n)
    out = []
    for k in range(a.steps):
        dj = D.to_device(-rng.uniform(0.1, 2.0, n))  # all negative: constraint active every step
        gv = float(x.mean()) - 0.4
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        x = mma_update(st, x, dj, gv, c, 1e-3, 1.0)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    print(json.dumps({"n": n, "mma_ms": out, "mean_x": float(x.mean())}))


if __name__ == "__main__":
    main()
