"""Timeline of a few steady-state pulses (engine event marks, SF_TRACE_FILE).
Usage: SF_PROFILE_GRAPHS=1 python tools/trace_pulses.py CONFIG [WARM] [TRACED]
Prints per-kind mean durations and the last pulses' intervals (us, relative)."""
import collections
import os
import sys
import tempfile

import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.geometry import pixel_positions  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1])]
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 32
traced = int(sys.argv[3]) if len(sys.argv) > 3 else 8
path = os.path.join(tempfile.mkdtemp(), "trace.txt")
os.environ["SF_TRACE_FILE"] = path
wl = generate(cfg, device_sim=True)
dev = torch.device("cuda", 0)
eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w,
             pixel_positions(wl.grid))
st = torch.cuda.current_stream(dev)
eng.set_stream(st)
g = torch.from_numpy(wl.positions).to(dev)
w = torch.from_numpy(wl.omega).to(dev)
d = torch.from_numpy(wl.d).to(dev)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device=dev)
c2 = torch.empty_like(c)
t = 1.0
for k in range(warm + traced):
    if k == warm:
        torch.cuda.synchronize()
        eng.profile(True)
    j = k % cfg.n_pulses
    eng.accumulate_geom(g[j], w, d[j], wl.sigma2)
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize()
eng.profile_read(0)
names = {0: "gemv", 1: "gram", 2: "loop", 3: "oper", 4: "lips", 5: "fista", 6: "ktilde",
         7: "fold"}
ev = collections.defaultdict(list)
for line in open(path):
    k, i, a, b = line.split()
    ev[int(k)].append((float(a), float(b)))
for k in sorted(ev):
    v = ev[k]
    print(f"{names[k]:7s} n={len(v):4d} mean {1e3 * sum(b - a for a, b in v) / len(v):8.1f} us")
starts = sorted(a for a, b in ev[5])
print("FISTA call periods (us):", [round(1e3 * (b - a)) for a, b in zip(starts, starts[1:])])
fi = sorted(ev[5])[-6:]
t0 = fi[0][0]
for k in sorted(ev):
    sel = [(round(1e3 * (a - t0)), round(1e3 * (b - t0))) for a, b in sorted(ev[k]) if b >= t0]
    print(names[k], sel[:14])
