"""Host-side time per pulse of the public-API loop (GeometricPulse -> accumulate ->
online_fista_pulse -> c_hat), by call, at a given result lag; B200."""
import collections
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2603_08582_b200 as api  # noqa: E402
from paper_2603_08582_b200.geometry import PulseGeometry  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
wl = generate(cfg)
M, n_r = wl.m_atoms, len(wl.omega)
pin_d = torch.from_numpy(np.ascontiguousarray(wl.d)).pin_memory()
pin_g = torch.from_numpy(np.ascontiguousarray(wl.positions)).pin_memory()
pin_w = torch.from_numpy(np.ascontiguousarray(wl.omega)).pin_memory()
stats = api.SufficientStatistics.empty(M, n_freq=n_r, dictionary=wl.dictionary, grid=wl.grid,
                                       mode="pixel")
state = api.SolverState(np.zeros(M), 1.0, stats)
sc = api.SolverConfig(lam_rel=cfg.lam_rel, inner_steps=cfg.steps)
cov = api.NoiseCovariance(sigma2=wl.sigma2)
acc = collections.defaultdict(float)


def one(k, lag, pending):
    global state
    t0 = time.perf_counter()
    j = k % cfg.n_pulses
    geo = PulseGeometry(j, pin_g[j].numpy(), pin_w.numpy())
    pulse = api.GeometricPulse(pin_d[j].numpy(), geo, cov, wl.grid, wl.dictionary)
    t1 = time.perf_counter()
    st2 = api.accumulate(state.stats, pulse)
    t2 = time.perf_counter()
    state = api.online_fista_pulse(api.SolverState(state.c_device(0), state.momentum_t, st2), sc)
    t3 = time.perf_counter()
    pending.append(state)
    while len(pending) > lag:
        float(pending.popleft().c_hat[0])
    t4 = time.perf_counter()
    acc["pulse objects"] += t1 - t0
    acc["accumulate"] += t2 - t1
    acc["online_fista_pulse"] += t3 - t2
    acc["c_hat read (wait)"] += t4 - t3


for lag in (1, 2, 4, 8, 16):
    pending = collections.deque()
    for k in range(20):
        one(k, lag, pending)
    while pending:
        float(pending.popleft().c_hat[0])
    torch.cuda.synchronize()
    acc.clear()
    n = 400
    t0 = time.perf_counter()
    for k in range(20, 20 + n):
        one(k, lag, pending)
    while pending:
        float(pending.popleft().c_hat[0])
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"lag {lag:2d}: {n / wall:8.1f} pulses/s  " +
          "  ".join(f"{k} {1e6 * v / n:6.1f} us" for k, v in acc.items()), flush=True)
