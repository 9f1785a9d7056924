"""Time FISTA calls alone (no concurrent pulse work) on a BASELINE config (GPU)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.geometry import pixel_positions  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
wl = generate(cfg)
eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w,
             pixel_positions(wl.grid))
for k in range(6):
    eng.accumulate_geom(wl.positions[k], wl.omega, wl.d[k], wl.sigma2)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device="cuda")
c2 = torch.empty_like(c)
t = 1.0
for k in range(5):
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
e0.record()
for k in range(n):
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
print(f"fista-only {cfg.name}: {ms * 1e3:.1f} us/call, {ms * 1e3 / cfg.steps:.2f} us/step")
