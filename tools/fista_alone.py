"""FISTA calls alone: after PULSES pulses of CONFIG, times repeated fista() calls on
the frozen state (no accumulate in between), next to the matvec alone.
Usage: python tools/fista_alone.py CONFIG PULSES [CALLS]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import CONFIGS, generate
cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2])
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 50
wl = generate(cfg, device_sim=True)
dev = torch.device("cuda", 0)
eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w, pixel_positions(wl.grid))
st = torch.cuda.current_stream(dev)
eng.set_stream(st)
g = torch.from_numpy(wl.positions).to(dev); w = torch.from_numpy(wl.omega).to(dev); d = torch.from_numpy(wl.d).to(dev)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device=dev); c2 = torch.empty_like(c)
t = 1.0
for k in range(n):
    eng.accumulate_geom(g[k % cfg.n_pulses], w, d[k % cfg.n_pulses], wl.sigma2)
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize()
c3 = torch.empty_like(c)
for _ in range(5):
    eng.fista(c, c3, cfg.steps, t, lam_rel=cfg.lam_rel)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(calls):
    eng.fista(c, c3, cfg.steps, t, lam_rel=cfg.lam_rel)
e1.record(st)
torch.cuda.synchronize()
us = 1e3 * e0.elapsed_time(e1) / calls
mv = eng.probe_matvec(20)
print(f"{cfg.name} after {n} pulses: fista call alone {us:.1f} us = {cfg.steps} x ({mv:.1f} matvec + "
      f"{(us - cfg.steps * mv) / cfg.steps:.1f} rest) us; nnz {int(torch.count_nonzero(c))}")
