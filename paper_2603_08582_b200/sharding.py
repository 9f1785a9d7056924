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


class PeerGroup:
    """Peer-memory exchange group (sf_peer_*): one process per GPU of one node,
    the ranks writing their partials straight into each other's device memory
    (CUDA IPC over NVLink) instead of calling a collective library.

    ``torch.distributed`` (any backend, gloo suffices) only carries the set-up:
    the name of the shared-memory block holding the ranks' sequence counters,
    and the ranks' IPC handle blobs."""

    def __init__(self, engine, rank, world, group=None):
        import torch.distributed as dist
        from multiprocessing import shared_memory

        self._lib = _lib.load()
        self.rank, self.world = int(rank), int(world)
        cy, ck = ctypes.c_int64(), ctypes.c_int64()
        check(self._lib.sf_shard_sizes(engine._h, ctypes.byref(cy), ctypes.byref(ck)))
        nbytes = 2 * 16 * 8
        if self.world > 1:
            name = [None]
            if self.rank == 0:
                self._shm = shared_memory.SharedMemory(create=True, size=nbytes)
                self._shm.buf[:nbytes] = bytes(nbytes)
                name[0] = self._shm.name
            dist.broadcast_object_list(name, src=0, group=group)
            if self.rank != 0:
                self._shm = shared_memory.SharedMemory(name=name[0])
                try:  # rank 0 owns the block: keep this process's tracker from unlinking it
                    from multiprocessing import resource_tracker

                    resource_tracker.unregister(self._shm._name, "shared_memory")
                except Exception:
                    pass
        else:
            self._shm = shared_memory.SharedMemory(create=True, size=nbytes)
            self._shm.buf[:nbytes] = bytes(nbytes)
        self._seq = (ctypes.c_uint64 * 32).from_buffer(self._shm.buf)
        h = ctypes.c_void_p()
        check(self._lib.sf_peer_create(int(engine.device), self.rank, self.world, cy.value,
                                       ck.value, ctypes.byref(self._seq), ctypes.byref(h)))
        self._h = h
        if self.world > 1:
            size = int(self._lib.sf_peer_blob_size())
            blob = ctypes.create_string_buffer(size)
            check(self._lib.sf_peer_export(self._h, blob))
            blobs = [None] * self.world
            dist.all_gather_object(blobs, blob.raw, group=group)
            check(self._lib.sf_peer_import(self._h, b"".join(blobs)))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.sf_peer_destroy(self._h)
            self._h = None
            del self._seq
            self._shm.close()
            if self.rank == 0:
                self._shm.unlink()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def shard_peer(engine, rank=None, world=None, group=None):
    """Shard ``engine`` over the ranks of a torch.distributed group with the
    peer-memory exchange; returns the PeerGroup (keep it alive with the engine)."""
    import torch.distributed as dist

    if rank is None or world is None:
        if dist.is_available() and dist.is_initialized():
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        else:
            rank, world = 0, 1
    pg = PeerGroup(engine, rank, world, group)
    check(_lib.load().sf_shard_init_peer(engine._h, pg._h))
    engine.rank, engine.world = int(rank), int(world)
    return pg


def shard_auto(engine, prefer="peer", group=None):
    """Shard ``engine`` over the torch.distributed ranks with the peer-memory
    exchange when every rank can set it up (IPC handles open, peer access), else
    with the NCCL all-reduces.  Returns ("peer", PeerGroup) or ("nccl", None);
    the decision is collective, so the ranks never disagree."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        shard_engine(engine, group=group)
        return "nccl", None
    pg, ok = None, 1
    if prefer == "peer":
        try:
            pg = PeerGroup(engine, dist.get_rank(group), dist.get_world_size(group), group)
        except Exception:  # any rank failing sends every rank to NCCL
            ok = 0
    else:
        ok = 0
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 1:
        check(_lib.load().sf_shard_init_peer(engine._h, pg._h))
        engine.rank, engine.world = pg.rank, pg.world
        return "peer", pg
    if pg is not None:
        pg.close()
    shard_engine(engine, group=group)
    return "nccl", None


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
