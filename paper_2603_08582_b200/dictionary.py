"""Edgelet dictionary (host, built once per run) and per-pulse composition.

Reference: dictionary.py:11-166.  The dictionary is kept as an ELL table
(atom j -> up to ``width`` (pixel, weight) pairs), the layout the device
compose kernel gathers from; the dense N x M matrix of the reference is only
materialised on request (``EdgeletDictionary.atoms``) for small problems.

Two builders:
  * ``build_dictionary(spec)``  -- the reference enumeration (dictionary.py:109-142):
    binary columns, atoms that lose a pixel to the border are dropped, exact
    duplicates removed.
  * ``build_extended_dictionary(...)`` -- the BASELINE.json dictionaries
    (SURVEY App. A G3): identity block + every (strided) origin per
    orientation, clipped atoms kept, columns normalised to unit 2-norm.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, ptr

_TWO_PI = 2.0 * math.pi


@dataclass
class EdgeletParams:
    """One atom: 1-pixel-wide segment with rotation, length, origin (dictionary.py:11-24)."""

    rotation: float
    length: int
    origin: tuple

    def __post_init__(self):
        self.rotation = float(self.rotation) % _TWO_PI
        self.length = int(self.length)
        self.origin = (int(self.origin[0]), int(self.origin[1]))
        if self.length < 1:
            raise ValueError("edgelet length must be at least 1")


@dataclass
class DictionarySpec:
    """Lengths x rotations to enumerate on a side x side grid (dictionary.py:27-48)."""

    lengths: tuple
    rotations: tuple
    side_pixels: int

    def __post_init__(self):
        side = int(self.side_pixels)
        if side < 2:
            raise ValueError("side_pixels must be at least 2")
        lengths = tuple(sorted({int(v) for v in self.lengths}))
        rotations = tuple(sorted({float(r) % _TWO_PI for r in self.rotations}))
        if not lengths or not rotations:
            raise ValueError("dictionary spec needs at least one length and one rotation")
        for ln in lengths:
            if ln < 1 or ln >= side:
                raise ValueError(f"edgelet length {ln} outside [1, {side - 1}]")
        self.lengths = lengths
        self.rotations = rotations
        self.side_pixels = side


@dataclass
class EdgeletDictionary:
    """ELL-form dictionary: ell_idx/ell_w are [m_atoms][width], index -1 = unused."""

    ell_idx: np.ndarray
    ell_w: np.ndarray
    n_pixels: int
    side_pixels: int = 0
    params: list = field(default_factory=list)
    _dense: np.ndarray = field(default=None, repr=False)

    @property
    def m_atoms(self):
        return self.ell_idx.shape[0]

    @property
    def atoms(self):
        """Dense N x M float64 matrix (reference EdgeletDictionary.atoms)."""
        if self._dense is None:
            H = np.zeros((self.n_pixels, self.m_atoms))
            j, l = np.nonzero(self.ell_idx >= 0)
            H[self.ell_idx[j, l], j] = self.ell_w[j, l]
            self._dense = H
        return self._dense


def _raster_pixels(rotation, length, x0, y0, side):
    """Pixels of one edgelet, clipped to the grid (stepping rule of dictionary.py:82-103)."""
    dx = math.cos(rotation)
    dy = math.sin(rotation)
    k = np.arange(length)
    if abs(dx) >= abs(dy):
        step = 1 if dx >= 0.0 else -1
        slope = dy / dx
        xs = x0 + step * k
        ys = np.floor(y0 + (step * k) * slope + 0.5).astype(np.int64)
    else:
        step = 1 if dy >= 0.0 else -1
        slope = dx / dy
        ys = y0 + step * k
        xs = np.floor(x0 + (step * k) * slope + 0.5).astype(np.int64)
    keep = (xs >= 0) & (xs < side) & (ys >= 0) & (ys < side)
    return (ys[keep] * side + xs[keep]).astype(np.int64)


def rasterize_edgelet(params, side_pixels):
    """Row-major 0/1 image of one edgelet, or None if fully clipped (dictionary.py:66-106)."""
    side = int(side_pixels)
    if side < 2:
        raise ValueError("side_pixels must be at least 2")
    if params.length >= side:
        raise ValueError("edgelet length must be below side_pixels")
    x0, y0 = params.origin
    if not (0 <= x0 < side and 0 <= y0 < side):
        raise ValueError("edgelet origin lies outside the grid")
    pix = _raster_pixels(params.rotation, params.length, x0, y0, side)
    if pix.size == 0:
        return None
    img = np.zeros(side * side)
    img[pix] = 1.0
    return img


def _to_ell(columns, n_pixels):
    width = max(len(c[0]) for c in columns)
    m = len(columns)
    idx = np.full((m, width), -1, dtype=np.int32)
    w = np.zeros((m, width), dtype=np.float64)
    for j, (p, v) in enumerate(columns):
        idx[j, :len(p)] = p
        w[j, :len(p)] = v
    return idx, w


def build_dictionary(spec, require_overcomplete=False):
    """Reference enumeration: rotation-major, then length, then origin (dictionary.py:109-142)."""
    side = spec.side_pixels
    columns, kept, seen = [], [], set()
    for rot in spec.rotations:
        for length in spec.lengths:
            for y in range(side):
                for x in range(side):
                    pix = _raster_pixels(rot, length, x, y, side)
                    uniq = np.unique(pix)
                    if uniq.size != length:  # lost a pixel to the border (dictionary.py:127)
                        continue
                    key = uniq.tobytes()
                    if key in seen:          # exact duplicate (dictionary.py:129-131)
                        continue
                    seen.add(key)
                    columns.append((uniq, np.ones(uniq.size)))
                    kept.append(EdgeletParams(rot, length, (x, y)))
    if not columns:
        raise ValueError("dictionary spec produced no atoms")
    n = side * side
    if require_overcomplete and len(columns) <= n:
        raise ValueError(f"dictionary is not over-complete: M={len(columns)} <= N={n}")
    idx, w = _to_ell(columns, n)
    return EdgeletDictionary(idx, w, n, side, kept)


def build_extended_dictionary(side, length, n_rotations, stride=1, identity=True):
    """BASELINE dictionaries.

    Column order: identity block (pixel order), then rotation-major, then origin
    row-major over the stride lattice.  Rotations are k * pi / n_rotations
    (4 -> 0, 45, 90, 135 deg; 8 -> multiples of 22.5 deg).  Clipped atoms are
    kept and every column is scaled to unit 2-norm (1/sqrt(pixel count)).
    """
    side = int(side)
    n = side * side
    rots = [k * math.pi / n_rotations for k in range(n_rotations)]
    columns, params = [], []
    if identity:
        for p in range(n):
            columns.append((np.array([p]), np.array([1.0])))
            params.append(None)
    for rot in rots:
        for y in range(0, side, stride):
            for x in range(0, side, stride):
                pix = np.unique(_raster_pixels(rot, length, x, y, side))
                columns.append((pix, np.full(pix.size, 1.0 / math.sqrt(pix.size))))
                params.append(EdgeletParams(rot, length, (x, y)))
    idx, w = _to_ell(columns, n)
    return EdgeletDictionary(idx, w, n, side, params)


def ell_from_dense(H):
    """ELL table of a dense N x M matrix (column nonzeros in pixel order)."""
    H = np.asarray(H, dtype=np.float64)
    if H.ndim != 2:
        raise ValueError("dictionary must be 2-d")
    nz = H != 0.0
    width = max(1, int(nz.sum(axis=0).max()) if H.size else 1)
    m = H.shape[1]
    idx = np.full((m, width), -1, dtype=np.int32)
    w = np.zeros((m, width))
    for j in range(m):
        p = np.nonzero(nz[:, j])[0]
        idx[j, :p.size] = p
        w[j, :p.size] = H[p, j]
    return idx, w


def _ell_of(dictionary):
    if isinstance(dictionary, EdgeletDictionary):
        return dictionary.ell_idx, dictionary.ell_w, dictionary.n_pixels
    H = np.asarray(dictionary)
    idx, w = ell_from_dense(H)
    return idx, w, H.shape[0]


def compose(forward, dictionary):
    """Per-pulse operator G = F H on the device (dictionary.py:151-157)."""
    F = np.ascontiguousarray(forward, dtype=np.complex128)
    idx, w, n = _ell_of(dictionary)
    if F.ndim != 2 or F.shape[1] != n:
        raise ValueError("incompatible operator shapes for compose")
    m = idx.shape[0]
    G = np.empty((F.shape[0], m), dtype=np.complex128)
    idx = np.ascontiguousarray(idx, dtype=np.int32)
    w = np.ascontiguousarray(w, dtype=np.float64)
    check(_lib.load().sf_compose_ell(0, ptr(F), F.shape[0], n, ptr(idx), ptr(w), m,
                                     idx.shape[1], ptr(G)))
    return G


def _transpose_ell(idx, w, n_pixels):
    """Pixel-major ELL (pixel -> atoms) of an atom-major table."""
    j, l = np.nonzero(idx >= 0)
    p = idx[j, l]
    order = np.lexsort((j, p))
    p, j, v = p[order], j[order], w[j[order], l[order]]
    counts = np.bincount(p, minlength=n_pixels)
    width = max(1, int(counts.max()) if counts.size else 1)
    tidx = np.full((n_pixels, width), -1, dtype=np.int32)
    tw = np.zeros((n_pixels, width))
    start = np.concatenate([[0], np.cumsum(counts)[:-1]])
    slot = np.arange(p.size) - start[p]
    tidx[p, slot] = j
    tw[p, slot] = v
    return tidx, tw


def synthesize(dictionary, coeffs):
    """Image H c (dictionary.py:160-166), on the device (compose of c^T with H^T)."""
    idx, w, n = _ell_of(dictionary)
    c = np.asarray(coeffs)
    if c.ndim != 1 or c.shape[0] != idx.shape[0]:
        raise ValueError("coefficient vector does not match atom count")
    tidx, tw = _transpose_ell(idx, w, n)
    row = np.ascontiguousarray(c.astype(np.complex128)[None, :])
    out = np.empty((1, n), dtype=np.complex128)
    check(_lib.load().sf_compose_ell(0, ptr(row), 1, idx.shape[0], ptr(tidx), ptr(tw), n,
                                     tidx.shape[1], ptr(out)))
    return out[0] if np.iscomplexobj(c) else out[0].real.copy()
