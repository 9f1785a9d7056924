"""Debug helper: geometric pulses of a golden fixture through the engine (GPU)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "tests")
sys.path.insert(0, ".")
from conftest import golden  # noqa: E402
import oracle.sarfista_oracle as orc  # noqa: E402
from paper_2603_08582_b200.engine import Engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "geom_small"
g = golden(name + ".npz")

m = g["ell_idx"].shape[0]
side = int(round(np.sqrt(g["image"].shape[0])))
eng = Engine(m, g["omega"].shape[0], g["ell_idx"], g["ell_w"], orc.pixel_positions(side))
for k in range(g["positions"].shape[0]):
    eng.accumulate_geom(g["positions"][k], g["omega"], g["d"][k], float(g["sigma2"][0]))
    torch.cuda.synchronize()
    print(k, eng.scalars(), eng.power_diag(), "ref L", g["L"][k])
