"""bench.py host logic without a GPU: the algorithmic byte model (DESIGN.md "Byte
model") and the reference arm's JSON contract."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    sys.path.insert(0, ROOT)
    import bench

    return bench


def test_byte_model_fp64_matches_survey():
    b = _bench()
    m, n, q = 2, 1000, 50
    # per element a2 a1 b2 b1 (32) + x r/w (16); per cell y + v r/w (24 / m); lo, hi per (i,k)
    # shared by q scenarios; ~11 row scalars per (i,j)
    per_elem = b.alg_bytes_per_iter(m, n, q) / (m * n * q)
    assert abs(per_elem - (32 + 16 + 24 / m + 16 / q + 88 / n)) < 1e-12
    assert 60.3 < per_elem < 60.5  # 60.3 B at m = 2, q >= 50


def test_byte_model_f2_fp32_coefficients():
    b = _bench()
    m, n, q = 2, 1000, 100000
    f64 = b.alg_bytes_per_iter(m, n, q, 64)
    f32 = b.alg_bytes_per_iter(m, n, q, 32)
    assert f64 - f32 == 16 * m * n * q  # four coefficient streams at 4 instead of 8 bytes
    assert abs(f32 / (m * n * q) - 44.0) < 0.1


def test_byte_model_horizon_m4():
    b = _bench()
    per_elem = b.alg_bytes_per_iter(4, 10**6, 1) / (4 * 10**6)
    assert 69.9 < per_elem < 70.1  # 70 B at m = 4, q = 1


def _reference_line(workload, steps="1", warmup="0"):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", workload, "--steps", steps, "--warmup", warmup],
                         capture_output=True, text=True, cwd=ROOT, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_prints_one_json_line():
    """--impl reference times the CPU oracle (the reference arm of this tier): one
    JSON line with impl=reference, the same metric/unit as our arm, e2e and
    cpu_baseline; no GPU needed."""
    d = _reference_line("toy")
    assert d["impl"] == "reference"
    assert d["unit"] == "element-updates/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"].startswith("oracle") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["cpu_count"] >= 1 and d["cpu_baseline"]["affinity"] >= 1


def test_reference_arm_default_workload_loads_no_product_code():
    """The default (headline) workload -- configs[3], q = 1e5 -- on the reference arm
    runs a bounded sample of scenario rows with q_total = 1e5, and the process never
    loads the product package or its CUDA library."""
    code = (
        "import sys, runpy, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "finally:\n"
        "    bad = [m for m in sys.modules if m.startswith('paper_1903_10041_b200')]\n"
        "    maps = open('/proc/self/maps').read()\n"
        "    print('LOADED', json.dumps(bad), 'libadmm_b200' in maps, file=sys.stderr)\n")
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                         env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    tail = [l for l in out.stderr.splitlines() if l.startswith("LOADED")][-1]
    assert tail == "LOADED [] False", tail
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["config"]["q_total"] == 100000 and d["config"]["baseline_config"] == "configs[3]"
    assert "q_total = 100000" in d["cpu_baseline"]["sample"]


def test_horizon_workload_blocks_at_n_gpus():
    """--workload horizon at N > 1 uses horizon blocks: rank r's problem is its balanced
    range [k0, k1) of the steps of the same synthetic instance (the slices tile the
    horizon), and the roofline's byte model counts the rank's own steps."""
    import argparse

    import numpy as np

    b = _bench()
    args = argparse.Namespace(workload="horizon", n=1001, q=None, family="C", coeff_bits=64)
    full = b.workload(args, 0, 1)["make"](0, 1)
    parts = []
    for r in range(3):
        W = b.workload(args, r, 3)
        assert W["horizon_blocks"] and W["scaling"] == "strong"
        P = W["make"](0, 1)
        assert P["n"] == W["k1"] - W["k0"] and P["a2"].shape == (4, 1, P["n"])
        parts.append(P)
    for key in ("a2", "b2", "b1"):
        assert np.array_equal(np.concatenate([p[key] for p in parts], axis=2), full[key])
    for key in ("lo", "hi", "y"):
        assert np.array_equal(np.concatenate([p[key] for p in parts], axis=1), full[key])


def test_reference_and_our_config_are_the_same_workload():
    """The driver compares the two arms' `config`: both are built by config_of from
    the same workload description (no engine / timing keys inside)."""
    import argparse

    b = _bench()
    args = argparse.Namespace(workload="toy", n=None, q=None, family="C", coeff_bits=64)
    W = b.workload(args, 0, 1)
    ref = _reference_line("toy")
    assert ref["config"] == b.config_of(args, W, 1)
