"""Late-regime matvec probe: runs CONFIG for PULSES pulses, then times the
matvec alone on the final iterate; prints the live-slab / live-row statistics
of the tiles.  Usage: python tools/sparse_probe.py CONFIG PULSES"""
import sys
import numpy as np
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
for k in range(n):
    j = k % cfg.n_pulses
    eng.accumulate_geom(g[j], w, d[j], wl.sigma2)
    t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
    c, c2 = c2, c
torch.cuda.synchronize()
print("nnz", int(torch.count_nonzero(c)), "matvec alone us", round(eng.probe_matvec(50), 2),
      "dense", round(eng.probe_matvec(50, dense=True), 2))
# support statistics from c: live pixels = union of the nonzero atoms' pixels
cn = c.cpu().numpy()
idx = wl.dictionary.ell_idx[np.nonzero(cn)[0]]
wts = wl.dictionary.ell_w[np.nonzero(cn)[0]]
pix = np.unique(idx[wts != 0])
npix = wl.grid.side_pixels ** 2
live = np.zeros(((npix + 127) // 128) * 128, bool); live[pix] = True
blk = live.reshape(-1, 128)
rows = blk.sum(1); slabs = blk.reshape(-1, 32, 4).any(2).sum(1)
nt = blk.shape[0]
print("live pixels", len(pix), "blocks with live", int((rows > 0).sum()), "of", nt)
print("rows/block: mean %.1f max %d; slabs/block mean %.1f max %d" % (rows.mean(), rows.max(), slabs.mean(), slabs.max()))
I, J = np.triu_indices(nt)
ns, nr = slabs[J], rows[I]
sparse = ns + nr // 2 <= 24
rounds = np.where(sparse, np.maximum((ns + 1) // 2, (nr + 3) // 4), 16)
print("tiles", len(I), "sparse", int(sparse.sum()), "rounds mean %.2f max %d" % (rounds.mean(), rounds.max()),
      "bytes MB %.1f" % ((np.where(sparse, ns * 2048 + nr * 512, 65536)).sum() / 1e6))
print("round histogram", np.bincount(rounds))
