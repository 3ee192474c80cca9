"""Host logic of bench.py (no GPU): the batch step's counter merge and the
threefold batch configuration (BASELINE.json configs[3])."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _fr(m, ms, launches):
    return {"matvecs": m, "startups": 1, "combines": 2, "terms": 3, "side": 495, "M": 13,
            "kernels": {"device_ms": ms, "gemm_ms": ms / 2, "gemm_launches": 7},
            "traffic": {"h2d_bytes": 10, "d2h_bytes": 4, "launches": launches},
            "times": {"tables": 0.5, "device": ms / 1e3}}


def test_merge_frobenius_sums_counters_and_keeps_shape():
    out = bench.merge_frobenius([_fr(100, 20.0, 5), _fr(50, 10.0, 3)])
    assert out["matvecs"] == 150 and out["startups"] == 2 and out["combines"] == 4 and out["terms"] == 6
    assert out["kernels"]["device_ms"] == 30.0 and out["kernels"]["gemm_launches"] == 14
    assert out["traffic"] == {"h2d_bytes": 20, "d2h_bytes": 8, "launches": 8}
    assert out["times"]["tables"] == 1.0
    assert out["side"] == 495 and out["M"] == 13


def test_threefold_batch_config():
    p, n, d, seed, desc = bench.CONFIGS["threefold_batch"]
    assert (p, n, d) == (13, 4, 3) and bench.BATCH_SEEDS == 64
    # ranks take seeds round-robin: every seed exactly once for any world size
    for world in (1, 2, 4, 8):
        got = sorted(s for r in range(world) for s in range(r, bench.BATCH_SEEDS, world))
        assert got == list(range(64))


def test_reference_arm_never_loads_the_product():
    """--impl reference runs the unmodified reference (oracle/_ref) only: the
    product package and libdrzg.so stay unloaded in that process"""
    import subprocess
    import pytest
    from conftest import have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json, bench\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'quintic', '--steps', '1', '--warmup', '0']\n"
            "bench.main()\n"
            "assert 'paper_2602_24155_b200' not in sys.modules\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libdrzg' not in maps, 'libdrzg.so mapped'\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["projection"] is False
