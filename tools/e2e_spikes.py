"""Per-pulse host wall time of the public-API loop right after engine creation
(finds one-off costs that fall into a short timed run).
Usage: python tools/e2e_spikes.py CONFIG [PULSES]"""
import collections
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200 import solver as api  # noqa: E402
from paper_2603_08582_b200.geometry import PulseGeometry  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
wl = generate(cfg, device_sim=True)
M = wl.m_atoms
pin_d = torch.from_numpy(np.ascontiguousarray(wl.d)).pin_memory()
pin_g = torch.from_numpy(np.ascontiguousarray(wl.positions)).pin_memory()
pin_w = torch.from_numpy(np.ascontiguousarray(wl.omega)).pin_memory()
stats = api.SufficientStatistics.empty(M, device=0, n_freq=cfg.n_freq, dictionary=wl.dictionary,
                                       grid=wl.grid)
state = api.SolverState(np.zeros(M), 1.0, stats)
sc = api.SolverConfig(lam_rel=cfg.lam_rel, inner_steps=cfg.steps)
cov = api.NoiseCovariance(sigma2=wl.sigma2)
pending = collections.deque()
ts = []
for k in range(n):
    t0 = time.perf_counter()
    geo = PulseGeometry(k, pin_g[k].numpy(), pin_w.numpy())
    pulse = api.GeometricPulse(pin_d[k].numpy(), geo, cov, wl.grid, wl.dictionary)
    st2 = api.accumulate(state.stats, pulse)
    t1 = time.perf_counter()
    state = api.online_fista_pulse(api.SolverState(state.c_device(0), state.momentum_t, st2), sc)
    t2 = time.perf_counter()
    pending.append(state)
    while len(pending) > 6:
        float(pending.popleft().c_hat[0])
    t3 = time.perf_counter()
    ts.append((1e6 * (t1 - t0), 1e6 * (t2 - t1), 1e6 * (t3 - t2)))
torch.cuda.synchronize()
for k, (a, b, c) in enumerate(ts):
    print(f"pulse {k:3d}: accumulate {a:8.0f} us  fista {b:8.0f} us  read {c:8.0f} us")
