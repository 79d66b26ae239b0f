"""The bench.py output contract on the CPU: `--impl reference` (the reference package's own CPU
path, composed from live phase rates) prints exactly one JSON line on stdout, with the keys the
driver reads.  Run at n = 16 (~10 s); skipped when the reference package is not installed."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _have_reference():
    return any(os.path.isdir(os.path.join(p, "gradfem"))
               for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"))


@pytest.mark.skipif(not _have_reference(), reason="reference package not installed")
def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--n", "16",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_bench_helpers():
    """In-solve roofline arithmetic and the partitioned allreduce count the bench line reports."""
    sys.path.insert(0, ROOT)
    import bench

    kprof = {"kernels_us": {"spmv_jacobi_r0": 500.0, "spmv_jacobi_tt": 480.0}}
    out = bench.jacobi_roofline(kprof, plain_bytes=2.7e9, rows=7.7e6, peak=6500.0)
    r0, tt = out["spmv_jacobi_r0"], out["spmv_jacobi_tt"]
    assert r0["bytes_per_launch"] == pytest.approx(2.7e9 + 16 * 7.7e6)  # + D^-1 and r0 rows
    assert tt["bytes_per_launch"] == pytest.approx(2.7e9 + 8 * 7.7e6)   # + D^-1 rows
    assert r0["achieved_gbs"] == pytest.approx(r0["bytes_per_launch"] / 500e-6 / 1e9)
    assert tt["frac"] == pytest.approx(tt["achieved_gbs"] / 6500.0)
    assert bench.jacobi_roofline(None, 1.0, 1.0, 1.0) is None
    env = os.environ.pop("B200FEM_DIST_FUSED_DOTS", None)
    try:
        assert [bench.dist_allreduces(n) for n in (1, 2, 3, 4, 8)] == [3, 3, 3, 2, 2]
        os.environ["B200FEM_DIST_FUSED_DOTS"] = "1"
        assert bench.dist_allreduces(1) == 2
        os.environ["B200FEM_DIST_FUSED_DOTS"] = "0"
        assert bench.dist_allreduces(8) == 3
    finally:
        os.environ.pop("B200FEM_DIST_FUSED_DOTS", None)
        if env is not None:
            os.environ["B200FEM_DIST_FUSED_DOTS"] = env
