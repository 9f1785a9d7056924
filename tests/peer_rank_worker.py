"""One rank of the two-process peer-memory exchange test (tests/test_peer_ranks.py).

Usage: python tests/peer_rank_worker.py RANK WORLD PORT OUT_NPZ N_PULSES
Both ranks use cuda:0 (the exchange has no kernel waiting on another rank, so
two processes may time-slice one device); gloo carries the set-up only."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

import sarfista_oracle as orc  # noqa: E402  (pixel positions only)
from paper_2603_08582_b200 import sharding  # noqa: E402
from paper_2603_08582_b200.dictionary import build_extended_dictionary  # noqa: E402
from paper_2603_08582_b200.engine import Engine  # noqa: E402
from paper_2603_08582_b200.workload import CONFIGS  # noqa: E402


def main():
    rank, world, port, out, n_pulses = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3],
                                        sys.argv[4], int(sys.argv[5]))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = dict(np.load(os.path.join(HERE, "golden", "oracle_cfg0.npz")))
    cfg = CONFIGS[0]
    dic = build_extended_dictionary(cfg.side, cfg.length, cfg.n_rot, cfg.stride)
    m = dic.m_atoms
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    eng = Engine(m, cfg.n_freq, dic.ell_idx, dic.ell_w, orc.pixel_positions(cfg.side))
    kind, pg = sharding.shard_auto(eng, prefer="peer")  # collective decision; NCCL if any rank fails
    assert kind == "peer", kind
    c = torch.zeros(m, dtype=torch.float64, device=dev)
    c2 = torch.empty_like(c)
    t = 1.0
    Ls = []
    for k in range(n_pulses):
        eng.accumulate_geom(g["positions"][k], g["omega"], g["d"][k], float(g["sigma2"][0]))
        t = eng.fista(c, c2, cfg.steps, t, lam_rel=cfg.lam_rel)
        c, c2 = c2, c
        Ls.append(eng.scalars()[0])
    np.savez(out, c=c.cpu().numpy(), t=t, L=np.array(Ls))
    dist.barrier()
    eng.close()
    pg.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
