"""Completion time of every grid (chain) of a C3 image (async, phase_log)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1509_06004_b200 import _native, synth
p = synth.generate(500, 375, 5, 5, rng_seed=0, types=("A", "B")).problems
s = _native.Solver(0, phase_log=1)
for r in range(2):
    s.solve_seed_batch(500, 375, p, synth.L20, "auto")
print("device ms", round(s.stats()["ms_device"], 2))
ends = []
t0 = None
import ctypes
raw = []
for g in range(len(p)):
    out = np.zeros(512, np.uint64); n = ctypes.c_int32(512)
    s._lib.pmf_debug_phases(s._h, g, out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(n))
    ts = (out[:n.value] & np.uint64((1 << 56) - 1)).astype(np.int64)
    raw.append((int(ts[0]), int(ts[-1]), n.value))
base = min(r[0] for r in raw)
ends = sorted((r[1] - base) / 1e3 for r in raw)
ends = [e / 1e3 for e in ends]
print("grid end times (ms): min %.1f p25 %.1f median %.1f p75 %.1f max %.1f" % (
    ends[0], np.percentile(ends, 25), np.median(ends), np.percentile(ends, 75), ends[-1]))
print("log entries per grid (capped at 511):", sorted(r[2] for r in raw)[-5:])
order = sorted(range(len(raw)), key=lambda g: raw[g][1])
slow = order[-3:]
print("slowest grids:", slow, "ends", [round((raw[g][1] - base) / 1e6, 1) for g in slow])
for g in slow[-1:]:
    s2 = _native.Solver(0)
    for r in range(2):
        s2.solve_seed_batch(500, 375, [p[g]], synth.L20, "auto")
    st = s2.stats()
    print("grid", g, "alone (cold per-lambda grids):", round(st["ms_device"], 2), "ms")
    s3 = _native.Solver(0, chain=20)
    for r in range(2):
        s3.solve_seed_batch(500, 375, [p[g]], synth.L20, "auto")
    print("grid", g, "alone as one warm chain:", round(s3.stats()["ms_device"], 2), "ms")
