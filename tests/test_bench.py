"""bench.py contract: the JSON line the driver parses (keys, units, consistency), the reference arm
(the oracle on the host cores) and the weak / strong workload shapes."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _line(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference times the oracle (this tier's reference) on a bounded sample and prints the
    same metric / unit with impl, cpu_baseline and a zero-byte e2e"""
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["metric"] == "zone-cycles/s" and d["unit"] == "zone-cycles/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.parametrize("strong", [False, True])
def test_workload_shapes(strong):
    """weak: 512^3 cells (512 blocks of 64^3) per GPU as one Morton cube per rank; strong: the 1-GPU mesh"""
    import bench
    import oracle as O
    for n in (1, 2, 4, 8):
        w = bench.workload("2b", n, strong=strong)
        cells = 1
        for d in range(3):
            cells *= w["mesh_nx"][d]
        assert w["block_nx"] == (64, 64, 64)
        assert cells == 512 ** 3 * (1 if strong else n)
        # unit cell width in every direction
        widths = {(w["xmax"][d] - w["xmin"][d]) / w["mesh_nx"][d] for d in range(3)}
        assert max(widths) - min(widths) < 1e-15
        nb = cells // 64 ** 3
        los = [O.partition(nb, n, r) for r in range(n)]
        assert all(hi - lo == nb // n for lo, hi in los)


@pytest.mark.gpu
def test_bench_line_on_gpu():
    """the N=1 headline line: metric / config / roofline / clocks / launches as the driver expects"""
    d = _line(["--steps", "2", "--warmup", "3", "--no-cpu"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["dtype"] == "f64" and d["scaling"] == "weak"
    assert d["value"] > 1e9 and abs(d["value"] - 512 ** 3 * 2 / (d["ms_per_step"] * 2e-3)) < 1e-6 * d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] < 1
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-12
    assert rf["fp64_pipe"]["bound"] == "alu" and 0 < rf["fp64_pipe"]["frac"] < 1
    assert d["gpu_launches"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
