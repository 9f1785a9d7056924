"""Debug helper: every scene of a batched engine vs single-scene engines (GPU)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import SMALL, generate_batch
name = sys.argv[1] if len(sys.argv) > 1 else "small8"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 5
scenes = generate_batch(SMALL[name], B); wl0 = scenes[0]
if len(sys.argv) > 3: scenes = scenes[::-1]
P = min(s.cfg.n_pulses for s in scenes)
mk = lambda b=1: Engine(wl0.m_atoms, len(wl0.omega), wl0.dictionary.ell_idx, wl0.dictionary.ell_w, pixel_positions(wl0.grid), batch=b)
eng = mk(B); singles = [mk() for _ in range(B)]
c = torch.zeros((B, wl0.m_atoms), dtype=torch.float64, device="cuda"); c2 = torch.empty_like(c)
cs = [torch.zeros(wl0.m_atoms, dtype=torch.float64, device="cuda") for _ in range(B)]; cs2 = [torch.empty_like(x) for x in cs]
t = 1.0; ts = [1.0] * B
for k in range(P):
    g = np.stack([s.positions[k] for s in scenes]); d = np.stack([s.d[k] for s in scenes]); s2 = np.array([s.sigma2 for s in scenes])
    eng.accumulate_geom_batch(g, wl0.omega, d, s2)
    t = eng.fista(c, c2, wl0.cfg.steps, t, lam_rel=wl0.cfg.lam_rel); c, c2 = c2, c
    Lb = eng.batch_scalars()[0]
    for b in range(B):
        e1 = singles[b]
        e1.accumulate_geom(scenes[b].positions[k], wl0.omega, scenes[b].d[k], scenes[b].sigma2)
        ts[b] = e1.fista(cs[b], cs2[b], wl0.cfg.steps, ts[b], lam_rel=wl0.cfg.lam_rel); cs[b], cs2[b] = cs2[b], cs[b]
        L1 = e1.scalars()[0]
        print(k, b, "L", Lb[b], L1, "L eq", Lb[b] == L1, "c eq", torch.equal(c[b], cs[b]), float((c[b] - cs[b]).abs().max()), "t", t == ts[b])
