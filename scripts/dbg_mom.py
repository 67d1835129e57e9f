import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from tests.test_gpu_momentum import run_momentum, random_plan, SEED, bits
import synthgen as sg
from oracle.momentum import weighted_f32, sequential_f64
from oracle.numerics import commits_from_plan
for gamma in (0.5, 0.9):
  for dt in (0, 1):
    rng = np.random.default_rng(int(gamma * 10) + dt)
    S = int(rng.choice([3, 8, 4099, 65_537, 200_003])); W = int(rng.integers(1, 20))
    p = random_plan(rng, W)
    (w, h, b, bh), h0 = run_momentum(S, W, dt, p, gamma)
    idx = np.arange(S)
    commits = commits_from_plan(p, lambda g: sg.update_values(SEED, g, 0, idx, dt))
    wr, hr, bk = weighted_f32(sg.w0_values(SEED, idx), h0, commits, 0.01, gamma, p["replica_boundary_commit"])
    dw = np.nonzero(bits(w) != bits(wr))[0]; dh = np.nonzero(bits(h) != bits(hr))[0]
    print(gamma, dt, S, W, p["commit_count"], "w mism", len(dw), dw[:6], "h mism", len(dh), dh[:6])
    for i in list(dw[:2]) + list(dh[:2]):
        print("  ", i, "w", w[i], wr[i], "h", h[i], hr[i], "h0", h0[i])
