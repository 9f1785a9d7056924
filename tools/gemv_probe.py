"""Run a BASELINE config's pulse stream, then launch the FISTA matvec alone on
the final state inside a cudaProfilerStart/Stop window (for
`ncu --profile-from-start off`): support-aware, then forced dense.
Usage: python tools/gemv_probe.py CONFIG [PULSES]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.geometry import pixel_positions  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_pulses
wl = generate(cfg, device_sim=True)
dev = torch.device("cuda", 0)
eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w,
             pixel_positions(wl.grid))
g = torch.from_numpy(wl.positions).to(dev)
w = torch.from_numpy(wl.omega).to(dev)
d = torch.from_numpy(wl.d).to(dev)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device=dev)
c2 = torch.empty_like(c)
t = 1.0
for k in range(n):
    j = k % cfg.n_pulses
    eng.accumulate_geom(g[j], w, d[j], wl.sigma2)
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize()
print("nnz(c)", int(torch.count_nonzero(c)), "alone us: sparse", eng.probe_matvec(20),
      "dense", eng.probe_matvec(20, dense=True))
torch.cuda.profiler.start()
eng.probe_matvec(1)
eng.probe_matvec(1, dense=True)
torch.cuda.profiler.stop()
