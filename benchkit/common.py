"""Shared bench plumbing: the metric string, the HBM peak, nvidia-smi clock sampling."""
from __future__ import annotations

import json
import os
import subprocess
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# BASELINE.json's metric, verbatim (the roofline fraction is the line's `roofline` object)
METRIC = "aggregated update GB/s committed (device-timed, max over ranks), % HBM/NVLink roofline"
HBM_FALLBACK = 6650.0


def hbm_peak():
    try:
        d = json.load(open(PEAKS))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line).

    start() launches the sampler (100 ms period) before the warm-up, because nvidia-smi takes a
    few hundred ms to print its first line and a short timed region would otherwise get none;
    mark() opens the timed window and __exit__ closes it; summary() keeps the samples whose
    nvidia-smi timestamp falls inside the window (widened by one sampling period at each end),
    else the nearest ones after the window opened (flagged)."""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def mark(self):
        self.t0 = time.time()

    def __enter__(self):
        if self.p is None:
            self.start()
        self.mark()
        return self

    def __exit__(self, *a):
        self.t1 = time.time()
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
            except ValueError:
                continue
        lo = (self.t0 or 0) - 0.1
        hi = (self.t1 or float("inf")) + 0.1
        win = [r for r in rows if lo <= r[0] <= hi]
        where = "timed window"
        if not win:
            win = [r for r in rows if r[0] >= lo][:2]
            where = "first samples after the timed window opened (window shorter than the sampler's start-up)"
        sm = sorted(r[1] for r in win)
        reasons = {nm for r in win for nm, v in zip(names, r[3]) if v.lower().startswith("active")}
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": win[-1][2] if win else None,
                "reasons": sorted(reasons), "samples": len(sm), "from": where}
