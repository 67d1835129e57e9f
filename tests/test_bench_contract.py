"""bench.py's JSON line keeps the driver's contract (keys, types, units)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    metric = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert BASE_KEYS <= set(d) and d["impl"] == "reference" and d["metric"] == metric
    assert d["unit"] == "GB/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "config2"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_gpu_line():
    d = _line(["--steps", "3", "--warmup", "3", "--no-variants", "--no-cpu-baseline"], 900)
    metric = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert BASE_KEYS <= set(d) and d["metric"] == metric and d["n_gpus"] == 1
    assert d["scaling"] == "weak" and d["data"] == "synthetic" and d["dtype"] == "f32"
    assert d["config"]["workload"] == "config2" and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] == d["steps"]                   # one fused commit per batch
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    e = d["e2e"]
    assert e["unit"] == "GB/s" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_clock_samples_are_taken_from_the_timed_window():
    """The clocks line keeps only nvidia-smi samples timestamped inside the timed window (widened
    by one 100 ms period); a window shorter than the sampler's start-up falls back to the first
    samples after it opened, and says so."""
    import datetime

    sys.path.insert(0, ROOT)
    from benchkit.common import Clocks

    def row(t, mhz, slow="Not Active", cap="Not Active"):
        ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return f"{ts}, 0, {mhz}, 1965, 700.0, 0x0, {slow}, Not Active, Not Active, {cap}"

    ck = Clocks(0)
    ck.t0, ck.t1 = 1000.0, 1001.0
    ck.lines = [row(999.5, 900, slow="Active"), row(1000.2, 1965), row(1000.5, 1950, cap="Active"),
                row(1000.8, 1965), row(1002.0, 800)]
    s = ck.summary()
    assert s["samples"] == 3 and s["sm_mhz"] == 1965.0 and s["reasons"] == ["sw_power_cap"]
    assert s["from"] == "timed window"
    ck.t0, ck.t1 = 1001.5, 1001.6                       # nothing inside: the next samples
    s = ck.summary()
    assert s["samples"] == 1 and s["sm_mhz"] == 800.0 and s["from"].startswith("first samples")
