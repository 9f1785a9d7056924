"""Checkpoint / resume of device-resident solver state (reference solver.py:302-369).

Two formats.
  * Statistics that keep the complex A (atom space, small M: the reference-API
    scale) are written in the reference's own text format -- a single file of
    hex floats, "sarfista-checkpoint 1", tags m / pulse_count / fallbacks /
    momentum_t / L / c_hat / b / one "A" line per row -- so checkpoints move
    between the reference and this engine in both directions, bit-exactly.
  * Everything else (pixel space, large M, sharded engines: complex A is 137 GB
    at cfg4) is a directory of binary arrays holding the engine's own state:
the packed fp32 tiles of the symmetric matrix (Re(A) in atom space, Re(B) in
pixel space), the fp64 vectors (b or beta, c_hat) and the scalars -- bit-exact,
and resuming continues identically (tests/test_gpu_parity.py).  A sharded
engine writes one ``tiles.rank<r>.npy`` per rank.
"""

import json
import os

import numpy as np

from ._lib import SF_MEM_HOST, check, ptr
from .solver import SolverState, SufficientStatistics

FORMAT = "sarfista-b200-checkpoint 1"
TEXT_MAGIC = "sarfista-checkpoint 1"


def _hex(values):
    return " ".join(float(v).hex() for v in values)


def _interleave(z):
    out = np.empty(2 * z.size)
    out[0::2] = z.real.ravel()
    out[1::2] = z.imag.ravel()
    return out


def save_text_checkpoint(path, state):
    """The reference's text format (solver.py:305-332) from device statistics."""
    stats = state.stats
    A = stats.A
    b = stats.b
    m = b.shape[0]
    lines = [TEXT_MAGIC, f"m {m}", f"pulse_count {stats.pulse_count}",
             f"fallbacks {stats.power_iteration_fallbacks}",
             "momentum_t " + float(state.momentum_t).hex(), "L " + float(stats.L).hex(),
             "c_hat " + _hex(np.asarray(state.c_hat, dtype=np.float64)),
             "b " + _hex(_interleave(b))]
    lines += ["A " + _hex(_interleave(A[i])) for i in range(m)]
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def load_text_checkpoint(path):
    """Parse the reference's text format (solver.py:335-369) into device statistics."""
    try:
        with open(path) as fh:
            lines = [ln.rstrip("\n") for ln in fh if ln.strip()]
    except UnicodeDecodeError:
        raise ValueError("not a recognizable checkpoint file") from None
    if not lines or lines[0] != TEXT_MAGIC:
        raise ValueError("not a recognizable checkpoint file")
    fields, rows = {}, []
    for ln in lines[1:]:
        tag, _, rest = ln.partition(" ")
        if tag == "A":
            rows.append(rest)
        else:
            fields[tag] = rest
    try:
        m = int(fields["m"])
        floats = lambda t: np.array([float.fromhex(x) for x in t.split()])  # noqa: E731
        c_hat = floats(fields["c_hat"])
        bb = floats(fields["b"])
        A = np.empty((m, m), dtype=np.complex128)
        if len(rows) != m or c_hat.shape != (m,) or bb.shape != (2 * m,):
            raise ValueError("checkpoint dimensions are inconsistent")
        for i, row in enumerate(rows):
            r = floats(row)
            if r.shape != (2 * m,):
                raise ValueError("checkpoint row length mismatch")
            A[i] = r[0::2] + 1j * r[1::2]
        stats = SufficientStatistics(A=A, b=bb[0::2] + 1j * bb[1::2], L=float.fromhex(fields["L"]),
                                     pulse_count=int(fields["pulse_count"]),
                                     power_iteration_fallbacks=int(fields["fallbacks"]))
        return SolverState(c_hat, float.fromhex(fields["momentum_t"]), stats)
    except KeyError as exc:
        raise ValueError(f"checkpoint lacks field {exc}") from None


def save_checkpoint(path, state):
    """Write ``state``: the reference text file when the statistics keep the
    complex A, else a directory of binary arrays."""
    stats = state.stats
    eng = stats.engine
    if eng is None or eng.keep_complex:
        return save_text_checkpoint(path, state)
    os.makedirs(path, exist_ok=True)
    L, n, fb, _ = eng.scalars()
    rank = getattr(eng, "rank", 0)
    world = getattr(eng, "world", 1)
    ij, tiles = eng.get_tiles()
    np.save(os.path.join(path, f"tiles.rank{rank}.npy"), tiles)
    np.save(os.path.join(path, f"tile_ij.rank{rank}.npy"), ij)
    if rank == 0:
        if eng.mode == "pixel":
            np.save(os.path.join(path, "beta.npy"), _pixel_beta(eng))
            np.save(os.path.join(path, "bp.npy"), eng.get_bp()[0])
        else:
            np.save(os.path.join(path, "b.npy"), eng.get_b())
        np.save(os.path.join(path, "c_hat.npy"), np.asarray(state.c_hat, dtype=np.float64))
        meta = {
            "format": FORMAT, "mode": eng.mode, "m_atoms": eng.m_atoms, "n_freq": eng.n_freq,
            "n_pixels": eng.n_pixels, "precision": eng.precision, "world": world,
            "L": float(L).hex(), "pulse_count": int(n), "fallbacks": int(fb),
            "momentum_t": float(state.momentum_t).hex(), "l_floor": float(stats.l_floor).hex(),
        }
        with open(os.path.join(path, "meta.json"), "w") as fh:
            json.dump(meta, fh, indent=1)


def _pixel_beta(eng):
    beta = np.empty(eng.n_pixels, dtype=np.complex128)
    check(eng._lib.sf_get_pixel_stats(eng._h, None, ptr(beta), SF_MEM_HOST))
    return beta


def load_checkpoint(path, dictionary=None, grid=None, device=0, rank=0, world=1, shard=None):
    """Rebuild a SolverState from ``path``.  Pixel-space checkpoints need the
    dictionary and grid the statistics were built with; ``shard`` is an optional
    callable(engine) applied before the state is restored (sharded resume)."""
    if os.path.isfile(path):
        return load_text_checkpoint(path)
    meta_path = os.path.join(path, "meta.json")
    if not os.path.exists(meta_path):
        raise ValueError("not a recognizable checkpoint directory")
    with open(meta_path) as fh:
        meta = json.load(fh)
    if meta.get("format") != FORMAT:
        raise ValueError("not a recognizable checkpoint directory")
    if meta["mode"] == "pixel":
        if dictionary is None or grid is None:
            raise ValueError("pixel-space checkpoints need the dictionary and grid")
        if dictionary.m_atoms != meta["m_atoms"] or grid.n_pixels != meta["n_pixels"]:
            raise ValueError(
                f"checkpoint holds statistics for {meta['m_atoms']} atoms over "
                f"{meta['n_pixels']} pixels; the dictionary has {dictionary.m_atoms} atoms "
                f"and the grid {grid.n_pixels} pixels")
    stats = SufficientStatistics(meta["m_atoms"], float.fromhex(meta["l_floor"]),
                                 precision=meta["precision"], device=device,
                                 n_freq=meta["n_freq"], dictionary=dictionary, grid=grid,
                                 mode=meta["mode"])
    eng = stats.engine
    if shard is not None:
        shard(eng)
    r = getattr(eng, "rank", rank)
    L = float.fromhex(meta["L"])
    if meta["mode"] == "pixel":
        beta = np.load(os.path.join(path, "beta.npy"))
        if beta.shape != (meta["n_pixels"],):
            raise ValueError("checkpoint beta does not match its pixel count")
        eng.set_pixel_stats(None, beta, L, meta["pulse_count"], meta["fallbacks"])
        bp_path = os.path.join(path, "bp.npy")
        if os.path.exists(bp_path):
            bp = np.ascontiguousarray(np.load(bp_path), dtype=np.complex128)
            if bp.shape != (meta["n_pixels"],):
                raise ValueError("checkpoint back-projection does not match its pixel count")
            check(eng._lib.sf_set_bp(eng._h, ptr(bp), SF_MEM_HOST))
    else:
        b = np.load(os.path.join(path, "b.npy"))
        if b.shape != (meta["m_atoms"],):
            raise ValueError("checkpoint b does not match its atom count")
        eng.set_stats(None, b, L, meta["pulse_count"], meta["fallbacks"])
    eng.set_tiles(np.load(os.path.join(path, f"tile_ij.rank{r}.npy")),
                  np.load(os.path.join(path, f"tiles.rank{r}.npy")))
    stats._version = eng.version
    c_hat = np.load(os.path.join(path, "c_hat.npy"))
    return SolverState(c_hat, float.fromhex(meta["momentum_t"]), stats)
