"""Run CONFIG for PULSES pulses, then 2 more inside a cudaProfilerStart/Stop window
(per-kernel launch list of a chosen regime: ncu --profile-from-start off).
Usage: python tools/window_launches.py CONFIG PULSES"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import CONFIGS, generate
cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2])
wl = generate(cfg, device_sim=True)
dev = torch.device("cuda", 0)
eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w, pixel_positions(wl.grid))
g = torch.from_numpy(wl.positions).to(dev); w = torch.from_numpy(wl.omega).to(dev); d = torch.from_numpy(wl.d).to(dev)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device=dev); c2 = torch.empty_like(c)
t = 1.0
for k in range(n + 2):
    if k == n:
        torch.cuda.synchronize(); torch.cuda.profiler.start()
    j = k % cfg.n_pulses
    eng.accumulate_geom(g[j], w, d[j], wl.sigma2)
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize(); torch.cuda.profiler.stop()
print("nnz", int(torch.count_nonzero(c)))
