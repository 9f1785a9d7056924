"""A/B helper: device-resident pulse rate of one BASELINE config with the
bench's loop (L2 flushed between pulses), for engine-knob experiments.
Usage: python tools/ab_pulse.py CONFIG [PULSES] [q]  (q: rate only; PRECISION=f16x3
selects the tensor-core Gram instead of the closed form)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.geometry import pixel_positions  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS, generate  # noqa: E402

cfg = CONFIGS[int(sys.argv[1])]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
wl = generate(cfg, device_sim=True)
dev = torch.device("cuda", 0)
import os  # noqa: E402

eng = Engine(wl.m_atoms, cfg.n_freq, wl.dictionary.ell_idx, wl.dictionary.ell_w,
             pixel_positions(wl.grid), precision=os.environ.get("PRECISION", "auto"),
             power_max_iter=int(os.environ.get("POWER_MAX_ITER", "0")))
st = torch.cuda.current_stream(dev)
eng.set_stream(st)
g = torch.from_numpy(wl.positions).to(dev)
w = torch.from_numpy(wl.omega).to(dev)
d = torch.from_numpy(wl.d).to(dev)
c = torch.zeros(wl.m_atoms, dtype=torch.float64, device=dev)
c2 = torch.empty_like(c)
flush = torch.empty(128 << 17, dtype=torch.float64, device=dev)
t = 1.0


def run(ks, t, c, c2):
    for k in ks:
        j = k % cfg.n_pulses
        eng.accumulate_geom(g[j], w, d[j], wl.sigma2)
        t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
        c, c2 = c2, c
        if not os.environ.get("NOFLUSH"):
            flush.fill_(float(k))
    return t, c, c2


start = int(os.environ.get("START", "8"))
t, c, c2 = run(range(start), t, c, c2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
t, c, c2 = run(range(start, start + n), t, c, c2)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{cfg.name} pulses/s {n / ms * 1e3:.1f} ({ms / n:.3f} ms/pulse)")
nz = int(torch.count_nonzero(c))
if len(sys.argv) > 3:
    sys.exit(0)
print(f"  final nnz(c) {nz}; matvec alone: support-aware {eng.probe_matvec(20):.1f} us, "
      f"dense {eng.probe_matvec(20, dense=True):.1f} us")
