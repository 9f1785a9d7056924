"""Tensor-core K~ vs the fp64 SIMT K~: per-pulse power-iteration results (GPU)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.geometry import pixel_positions  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 0]
npulse = int(sys.argv[2]) if len(sys.argv) > 2 else 6
wl = generate(cfg)
res = {}
for v in ("0", "1"):
    os.environ["SF_KTILDE_TC"] = v
    eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w,
                 pixel_positions(wl.grid))
    c = torch.zeros(wl.m_atoms, dtype=torch.float64, device="cuda")
    c2 = torch.empty_like(c)
    t = 1.0
    diags = []
    for k in range(npulse):
        eng.accumulate_geom(wl.positions[k], wl.omega, wl.d[k], wl.sigma2)
        t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
        c, c2 = c2, c
        torch.cuda.synchronize()
        diags.append(eng.power_diag())
    res[v] = (diags, eng.scalars(), c.cpu().numpy())
for k in range(npulse):
    a, b = res["0"][0][k], res["1"][0][k]
    print(k, "inc %.12e %.12e rel %.2e" % (a[0], b[0], abs(a[0] - b[0]) / abs(a[0])),
          "it", a[1], b[1], "frob rel %.2e" % (abs(a[3] - b[3]) / abs(a[3])))
c0, c1 = res["0"][2], res["1"][2]
print("L", res["0"][1][0], res["1"][1][0], "c rel", np.linalg.norm(c1 - c0) / max(np.linalg.norm(c0), 1e-300))
