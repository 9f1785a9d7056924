"""cProfile of the end-to-end API loop (GeometricPulse -> accumulate -> FISTA -> c_hat)."""
import cProfile
import pstats
import sys

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


def one(k):
    global state
    j = k % cfg.n_pulses
    geo = PulseGeometry(j, pin_g[j].numpy(), pin_w.numpy())
    pulse = api.GeometricPulse(pin_d[j].numpy(), geo, cov, wl.grid, wl.dictionary)
    st2 = api.accumulate(state.stats, pulse)
    prev = state
    state = api.online_fista_pulse(api.SolverState(state.c_device(0), state.momentum_t, st2), sc)
    return float(prev.c_hat[0])


for k in range(20):
    one(k)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for k in range(20, 220):
    one(k)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
