"""CPU: the shard planner and the sharded FISTA exchange pattern (gloo, 2 ranks).

The product's planner (sf_plan_shard, host-only C) is called through ctypes;
the two-rank test reproduces the engine's decomposition -- each rank applies
only its own tiles of the stored triangle (diagonal tiles through their upper
triangle), one all-reduce of the partial y_pix per step, the element-wise step
redundantly -- and must match the unsharded float64 FISTA loop of the oracle.
"""

import os
import socket

import numpy as np
import pytest

from paper_2603_08582_b200 import sharding

T = 128


def items_of(nt):
    ns = (nt + 1) // 2
    return [(a, b) for a in range(ns) for b in range(a, ns)]


def tiles_of_item(it, nt):
    out = []
    for a in range(2):
        for b in range(2):
            I, J = 2 * it[0] + a, 2 * it[1] + b
            if I >= nt or J >= nt or (it[0] == it[1] and a == 1 and b == 0):
                continue
            out.append((I, J))
    return out


@pytest.mark.parametrize("n_dim", [1, 128, 300, 1024, 4096, 16384, 65536])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_plan_partitions_every_tile_once(n_dim, world):
    nt = (n_dim + T - 1) // T
    items = items_of(nt)
    parts = sharding.plan(n_dim, world)
    assert parts[0][0] == 0 and parts[-1][1] == len(items)
    for (a0, a1, _), (b0, _, _) in zip(parts, parts[1:]):
        assert a1 == b0
    seen = []
    for i0, i1, nl in parts:
        tl = [t for k in range(i0, i1) for t in tiles_of_item(items[k], nt)]
        assert len(tl) == nl
        seen += tl
    total = nt * (nt + 1) // 2
    assert sorted(seen) == sorted((I, J) for I in range(nt) for J in range(I, nt))
    if total >= 8 * world:  # balanced to within one super-tile (4 tiles)
        counts = [p[2] for p in parts]
        assert max(counts) - min(counts) <= 4 + total // (4 * world * world) + 4


def local_matvec(S, x, tiles, n):
    """Partial y = S x over `tiles` with the engine's symmetric-store semantics."""
    y = np.zeros(n)
    for I, J in tiles:
        r0, c0 = I * T, J * T
        blk = S[r0:r0 + T, c0:c0 + T]
        if I == J:
            up = np.triu(blk)
            y[r0:r0 + T] += up @ x[c0:c0 + T]
            y[c0:c0 + T] += np.triu(blk, 1).T @ x[r0:r0 + T]
        else:
            y[r0:r0 + T] += blk @ x[c0:c0 + T]
            y[c0:c0 + T] += blk.T @ x[r0:r0 + T]
    return y


def problem(seed=3, n=300, m=420):
    rng = np.random.default_rng(seed)
    npad = (n + T - 1) // T * T
    Bm = rng.standard_normal((n, 40))
    S = np.zeros((npad, npad))
    S[:n, :n] = Bm @ Bm.T / 40 + 0.1 * np.eye(n)
    H = np.zeros((n, m))
    for j in range(m):
        px = rng.choice(n, size=rng.integers(1, 5), replace=False)
        H[px, j] = 1.0 / np.sqrt(px.size)
    breal = rng.standard_normal(m)
    return S, H, breal, npad, n


def fista_sharded(S, H, breal, npad, n, steps, rank, world, allreduce):
    nt = npad // T
    i0, i1, _ = sharding.plan(npad, world)[rank]
    items = items_of(nt)
    tiles = [t for k in range(i0, i1) for t in tiles_of_item(items[k], nt)]
    m = H.shape[1]
    A_norm = np.linalg.norm(H.T @ S[:n, :n] @ H, 2)
    tau, thresh = 1.0 / A_norm, 0.05 / A_norm
    z = np.zeros(m)
    cprev = z.copy()
    t = 1.0
    for _ in range(steps):
        x = np.zeros(npad)
        x[:n] = H @ z
        y = allreduce(local_matvec(S, x, tiles, npad))
        g = H.T @ y[:n] - breal
        u = z - tau * g
        c = np.sign(u) * np.maximum(np.abs(u) - thresh, 0.0)
        t_next = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        z = c + ((t - 1.0) / t_next) * (c - cprev)
        cprev, t = c, t_next
    return cprev, tau, thresh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, steps, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S, H, breal, npad, n = problem()

    def allreduce(v):
        tv = torch.from_numpy(v.copy())
        dist.all_reduce(tv)
        return tv.numpy()

    c, _, _ = fista_sharded(S, H, breal, npad, n, steps, rank, world, allreduce)
    out[rank] = c.tolist()
    dist.destroy_process_group()


def test_two_rank_sharded_fista_matches_unsharded():
    import sys
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle"))
    import sarfista_oracle as orc

    steps = 12
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), steps, out), nprocs=2, join=True)
    S, H, breal, npad, n = problem()
    _, tau, thresh = fista_sharded(S, H, breal, npad, n, 1, 0, 1, lambda v: v)
    A = H.T @ S[:n, :n] @ H
    ref, _ = orc.fista_inner(A, breal, np.zeros(H.shape[1]), 1.0, tau, thresh, steps)
    for r in range(2):
        c = np.array(out[r])
        assert np.linalg.norm(c - ref) <= 1e-11 * np.linalg.norm(ref)
    assert out[0] == out[1]  # identical on every rank after the all-reduce
