"""Debug helper: per-scene pulse buffers, batched vs single engine (GPU)."""
import ctypes, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2603_08582_b200 import _lib
from paper_2603_08582_b200.engine import Engine
from paper_2603_08582_b200.geometry import pixel_positions
from paper_2603_08582_b200.workload import SMALL, generate_batch
name, B, sc = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
scenes = generate_batch(SMALL[name], B); wl0 = scenes[0]
lib = _lib.load()
def buf(e, what, s, n):
    out = np.zeros(n)
    _lib.check(lib.sf_debug_pulse_buffer(e._h, what, s, out.ctypes.data_as(ctypes.c_void_p)))
    return out
eng = Engine(wl0.m_atoms, len(wl0.omega), wl0.dictionary.ell_idx, wl0.dictionary.ell_w, pixel_positions(wl0.grid), batch=B)
e1 = Engine(wl0.m_atoms, len(wl0.omega), wl0.dictionary.ell_idx, wl0.dictionary.ell_w, pixel_positions(wl0.grid))
g = np.stack([s.positions[0] for s in scenes]); d = np.stack([s.d[0] for s in scenes]); s2 = np.array([s.sigma2 for s in scenes])
eng.accumulate_geom_batch(g, wl0.omega, d, s2)
e1.accumulate_geom(scenes[sc].positions[0], wl0.omega, scenes[sc].d[0], scenes[sc].sigma2)
nr = len(wl0.omega); n = wl0.grid.n_pixels
for what, cnt, nm in ((4, 0, "in"), (3, 2 * n, "dbeta"), (1, 2 * nr, "u0"), (0, 2 * nr * nr, "K"), (2, 8, "pdiag")):
    if what == 4:
        continue
    a, b = buf(eng, what, sc, cnt), buf(e1, what, 0, cnt)
    print(nm, np.array_equal(a, b), np.abs(a - b).max(), np.argmax(np.abs(a - b)))
