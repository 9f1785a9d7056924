"""One scene's pixel-space statistics sharded over several GPUs.

The engine splits the Gram work items (2x2 super-tiles of the stored
triangle) into contiguous tile-balanced ranges (``sf_plan_shard``); each rank
updates and multiplies with its own tiles, and every FISTA step sums the
partial ``y_pix = Re(B) x`` over ranks with one NCCL all-reduce inside the
engine.  ``torch.distributed`` is only the plumbing that hands rank 0's NCCL
unique id to the other ranks.
"""

import ctypes

from . import _lib
from ._lib import check


def plan(n_dim, world):
    """[(item_begin, item_end, local_tiles)] per rank for a D x D symmetric store."""
    lib = _lib.load()
    out = []
    for r in range(world):
        i0, i1, nl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(lib.sf_plan_shard(int(n_dim), r, int(world), ctypes.byref(i0), ctypes.byref(i1),
                                ctypes.byref(nl)))
        out.append((i0.value, i1.value, nl.value))
    return out


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    check(_lib.load().sf_nccl_unique_id(buf))
    return buf.raw


class LoopbackGroup:
    """Emulated ranks on one device (sf_loopback_create): engines sharded into
    this group exchange through device slots and host barriers instead of NCCL.
    Each engine must be driven by its own host thread, the threads in lockstep
    (every accumulate / fista call of one rank matched by the others)."""

    def __init__(self, world):
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        check(self._lib.sf_loopback_create(int(world), ctypes.byref(h)))
        self._h = h
        self.world = int(world)

    def close(self):
        if self._h:
            self._lib.sf_loopback_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def shard_loopback(engine, rank, group):
    """Shard ``engine`` as rank ``rank`` of a LoopbackGroup."""
    check(_lib.load().sf_shard_init_loopback(engine._h, int(rank), group._h))
    return engine


def shard_engine(engine, rank=None, world=None, group=None):
    """Shard ``engine`` over the ranks of a torch.distributed group (or a single
    rank when no process group is initialised)."""
    import torch.distributed as dist

    if rank is None or world is None:
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
    uid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = obj[0]
    engine.shard(rank, world, uid)
    return engine
