"""The reference's plugin seam (kernels.py:27-116), served by the device library.

``delay_phase_matrix`` and ``fista_inner`` keep the reference signatures and
value semantics (inputs never mutated, new arrays returned).  There is one
implementation -- the sm_100a kernels -- so the reference's import-time
numpy/numba dispatch (kernels.py:56-116) has no counterpart here.
"""

import ctypes

import numpy as np

from . import _lib
from ._lib import check, ptr

DEVICE = 0


def delay_phase_matrix(omegas, delays):
    """Entry (m, i) = exp(-j omegas[m] delays[i]) (kernels.py:27-29, 66-76)."""
    w = np.ascontiguousarray(omegas, dtype=np.float64)
    t = np.ascontiguousarray(delays, dtype=np.float64)
    if w.ndim != 1 or t.ndim != 1:
        raise ValueError("omegas and delays must be 1-d")
    out = np.empty((w.shape[0], t.shape[0]), dtype=np.complex128)
    check(_lib.load().sf_delay_phase_matrix(DEVICE, ptr(w), w.shape[0], ptr(t), t.shape[0],
                                            ptr(out)))
    return out


def fista_inner(gram_re, corr_re, c0, t0, tau, thresh, steps):
    """``steps`` FISTA iterations on (gram_re, corr_re) from c0 (kernels.py:32-53, 78-103).

    Returns (c_last, t).  The matrix is packed to fp32 tiles on the device
    (upper triangle only when it is exactly symmetric); vectors stay fp64.
    """
    g = np.ascontiguousarray(gram_re, dtype=np.float64)
    b = np.ascontiguousarray(corr_re, dtype=np.float64)
    c = np.ascontiguousarray(c0, dtype=np.float64)
    m = c.shape[0]
    if g.shape != (m, m) or b.shape != (m,):
        raise ValueError("gram_re must be m x m and corr_re length m")
    out = np.empty(m, dtype=np.float64)
    t = ctypes.c_double()
    check(_lib.load().sf_fista_inner(DEVICE, ptr(g), ptr(b), ptr(c), m, float(t0), float(tau),
                                     float(thresh), int(steps), ptr(out), ctypes.byref(t)))
    return out, t.value
