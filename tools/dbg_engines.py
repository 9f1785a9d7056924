"""Debug helper: N single-scene engines fed identical pulses must agree bitwise (GPU)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import SMALL, generate_batch
wl = generate_batch(SMALL["small8"], 1)[0]
N = int(sys.argv[1]) if len(sys.argv) > 1 else 7
engs = [Engine(wl.m_atoms, len(wl.omega), wl.dictionary.ell_idx, wl.dictionary.ell_w, pixel_positions(wl.grid)) for _ in range(N)]
for k in range(3):
    for e in engs:
        e.accumulate_geom(wl.positions[k], wl.omega, wl.d[k], wl.sigma2)
    Ls = [e.scalars()[0] for e in engs]
    print(k, [L == Ls[0] for L in Ls], [e.power_diag()[1] for e in engs])
