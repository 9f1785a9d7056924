"""Float64 CPU oracle for the Online-FISTA per-pulse hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this module;
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may use it, and only as the checker or the timed CPU
baseline.

It restates, in numpy float64, the reference package ``sarfista``
(pkg/src/sarfista/ under the reference tree) line by line:

  splitmix64 / counter_uniform / counter_unit_complex_vector   rng.py:14-37
  pixel_positions                                               scene.py:93-105
  angular_frequencies, trajectory, platform_position            geometry.py:50-90
  forward_matrix (tau, exp(-j w tau))                           geometry.py:97-107, kernels.py:27-29
  compose G = F H with H as ELL (sparse)                        dictionary.py:151-157
  accumulate: Re(A) += Re(G^H R^-1 G) (+ optional complex A),   solver.py:178-206
              b += G^H R^-1 d, L += lambda_max(dA) with fallback
  hermitian_top_eigenvalue (M-space, literal)                   solver.py:139-175
  top eigenvalue in N_r space (identical iterate sequence)
  fista_inner                                                   kernels.py:32-53
  online_fista_pulse                                            solver.py:209-226
  reconstruct                                                   solver.py:294-299

Parity pins: tests/golden/*.npz were produced by the reference itself
(tests/golden/make_golden.py) and tests/test_oracle.py checks this module
against every one of them plus the reference's known-answer values.
"""

import math

import numpy as np
from scipy.linalg import blas as _blas

SPEED_OF_LIGHT = 299_792_458.0
_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15


# --- rng.py:14-37 ---------------------------------------------------------------
def splitmix64(state):
    z = (int(state) + _GOLDEN) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return (z ^ (z >> 31)) & _MASK


def counter_uniform(seed, index):
    mixed = splitmix64(((seed & _MASK) * _GOLDEN + index + 1) & _MASK)
    return (mixed >> 11) * 2.0 ** -53


def counter_unit_complex_vector(n, salt=0x5EED):
    """Vectorised restatement (uint64 wraparound) of rng.py:28-37."""
    k = np.arange(int(n), dtype=np.uint64)
    g = np.uint64(_GOLDEN)
    with np.errstate(over="ignore"):
        def mix(z):
            z = z + g
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return z ^ (z >> np.uint64(31))

        base = np.uint64(salt) * g + np.uint64(1)
        u_re = (mix(base + np.uint64(2) * k) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u_im = (mix(base + np.uint64(2) * k + np.uint64(1)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    v = (u_re - 0.5) + 1j * (u_im - 0.5)
    nrm = np.linalg.norm(v)
    if nrm == 0.0:
        v = np.ones(int(n), dtype=np.complex128)
        nrm = math.sqrt(float(n))
    return v / nrm


# --- scene.py / geometry.py -------------------------------------------------------
def pixel_positions(side, spacing=1.0, center=(0.0, 0.0, 0.0)):
    half = 0.5 * (side - 1)
    cx, cy, cz = center
    cols = np.tile(np.arange(side), side)
    rows = np.repeat(np.arange(side), side)
    out = np.empty((side * side, 3))
    out[:, 0] = cx + (cols - half) * spacing
    out[:, 1] = cy + (half - rows) * spacing
    out[:, 2] = cz
    return out


def angular_frequencies(n, center_hz, bandwidth_hz):
    if n == 1:
        return np.array([2.0 * math.pi * center_hz])
    f = np.linspace(center_hz - 0.5 * bandwidth_hz, center_hz + 0.5 * bandwidth_hz, n)
    return 2.0 * math.pi * f


def platform_position(radius, altitude, arc_start, arc_end, num_positions, center, k):
    if num_positions == 1:
        theta = arc_start
    else:
        theta = arc_start + (k / (num_positions - 1)) * (arc_end - arc_start)
    cx, cy, cz = center
    return np.array([cx + radius * math.cos(theta), cy + radius * math.sin(theta), cz + altitude])


def delays(gamma, xyz):
    diff = xyz - np.asarray(gamma, dtype=np.float64)[None, :]
    dists = np.sqrt((diff * diff).sum(axis=1))
    if np.any(dists == 0.0):
        raise ValueError("platform position coincides with a scene pixel")
    return (2.0 / SPEED_OF_LIGHT) * dists


def delay_phase_matrix(omegas, tau):
    return np.exp(-1j * np.outer(omegas, tau))


def forward_matrix(omega, gamma, xyz):
    return delay_phase_matrix(omega, delays(gamma, xyz))


def compose_ell(F, ell_idx, ell_w):
    """G[:, j] = sum_l w_jl F[:, idx_jl] (dense complex F @ sparse H)."""
    m, width = ell_idx.shape
    G = np.zeros((F.shape[0], m), dtype=np.complex128)
    for l in range(width):
        idx = ell_idx[:, l]
        ok = idx >= 0
        G[:, ok] += F[:, idx[ok]] * ell_w[ok, l][None, :]
    return G


def dense_from_ell(ell_idx, ell_w, n):
    H = np.zeros((n, ell_idx.shape[0]))
    j, l = np.nonzero(ell_idx >= 0)
    H[ell_idx[j, l], j] = ell_w[j, l]
    return H


# --- solver.py:139-175 ---------------------------------------------------------------
def hermitian_top_eigenvalue(X, rel_tol=1e-6, max_iter=500):
    X = np.asarray(X)
    v = counter_unit_complex_vector(X.shape[0])
    lam_prev = None
    delta_prev = None
    for _ in range(int(max_iter)):
        w = X @ v
        lam = float(np.real(np.vdot(v, w)))
        norm_w = float(np.linalg.norm(w))
        if norm_w == 0.0:
            return 0.0, True
        v = w / norm_w
        if lam_prev is not None:
            delta = lam - lam_prev
            if abs(delta) <= rel_tol * max(abs(lam), 1e-300):
                tail = 0.0
                if delta_prev is not None and abs(delta_prev) > abs(delta) > 0.0:
                    q = delta / delta_prev
                    if 0.0 < q < 1.0:
                        tail = delta * q / (1.0 - q)
                return lam + tail + abs(delta), True
            delta_prev = delta
        lam_prev = lam
    return (lam_prev if lam_prev is not None else 0.0), False


def top_eigenvalue_nr(Gw, v0, rel_tol=1e-6, max_iter=500):
    """Same iterate sequence as hermitian_top_eigenvalue(Gw^H Gw) with start v0,
    carried in the N_r-dimensional image u = Gw v."""
    K = Gw @ Gw.conj().T
    u = Gw @ v0
    lam_prev = None
    delta_prev = None
    it = 0
    for it in range(int(max_iter)):
        lam = float(np.real(np.vdot(u, u)))
        Ku = K @ u
        norm_w = math.sqrt(max(float(np.real(np.vdot(u, Ku))), 0.0))
        if norm_w == 0.0:
            return 0.0, True, it + 1, K
        u = Ku / norm_w
        if lam_prev is not None:
            delta = lam - lam_prev
            if abs(delta) <= rel_tol * max(abs(lam), 1e-300):
                tail = 0.0
                if delta_prev is not None and abs(delta_prev) > abs(delta) > 0.0:
                    q = delta / delta_prev
                    if 0.0 < q < 1.0:
                        tail = delta * q / (1.0 - q)
                return lam + tail + abs(delta), True, it + 1, K
            delta_prev = delta
        lam_prev = lam
    return (lam_prev if lam_prev is not None else 0.0), False, it + 1, K


# --- kernels.py:32-53 ------------------------------------------------------------------
def fista_inner(gram_re, corr_re, c0, t0, tau, thresh, steps):
    return fista_loop(lambda z: gram_re @ z, corr_re, c0, t0, tau, thresh, steps)


def fista_loop(matvec, corr_re, c0, t0, tau, thresh, steps):
    c_prev = np.array(c0, dtype=np.float64)
    z = c_prev.copy()
    t = t0
    for _ in range(steps):
        g = matvec(z) - corr_re
        u = z - tau * g
        c = np.sign(u) * np.maximum(np.abs(u) - thresh, 0.0)
        t_next = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t * t))
        z = c + ((t - 1.0) / t_next) * (c - c_prev)
        c_prev = c
        t = t_next
    return c_prev, t


# --- solver.py:88-226 -----------------------------------------------------------------
class OracleStats:
    """(Re A, b, L, n, fallbacks); optionally the full complex A for small M.

    Re(A) is held as the upper triangle of a Fortran-ordered float64 matrix and
    updated with BLAS dsyrk (A += P^T P, P = [Re G~; Im G~]), read by dsymv in
    the FISTA loop.  The rank update is then exactly symmetric, so the
    reference's symmetrisations (solver.py:181, 193) are identities here;
    ``A_re`` returns the full symmetric matrix."""

    def __init__(self, m, l_floor=1e-12, keep_complex=False):
        self._Au = np.zeros((m, m), order="F")
        self.A = np.zeros((m, m), dtype=np.complex128) if keep_complex else None
        self.b = np.zeros(m, dtype=np.complex128)
        self.L = float(l_floor)
        self.pulse_count = 0
        self.fallbacks = 0
        self.last_power = None
        self._v0 = None

    @property
    def A_re(self):
        u = np.triu(self._Au)
        return u + np.triu(u, 1).T

    def matvec(self, z):
        return _blas.dsymv(1.0, self._Au, z, lower=0)

    def v0(self):
        if self._v0 is None:
            self._v0 = counter_unit_complex_vector(self.b.shape[0])
        return self._v0


def whiten(G, d, sigma2=None, R=None):
    """Scalar sigma^2 or a full covariance -> (G~, d~) with dA = G~^H G~ (solver.py:178-183)."""
    if R is None:
        s = 1.0 / math.sqrt(sigma2)
        return G * s, d * s
    w, U = np.linalg.eigh(np.asarray(R, dtype=np.complex128))
    inv_sqrt = (U / np.sqrt(w)) @ U.conj().T
    return inv_sqrt @ G, inv_sqrt @ d


def accumulate(stats, G, d, sigma2=None, R=None, literal_power=False, fallback_hook=None):
    Gw, dw = whiten(np.asarray(G, dtype=np.complex128), np.asarray(d, dtype=np.complex128),
                    sigma2, R)
    P = np.ascontiguousarray(np.concatenate([Gw.real, Gw.imag], axis=0), dtype=np.float64)
    # A_re (upper) += P^T P  (Re(G^H G) = Gr^T Gr + Gi^T Gi)
    _blas.dsyrk(1.0, np.asfortranarray(P), beta=1.0, c=stats._Au, trans=1, lower=0,
                overwrite_c=1)
    if stats.A is not None:
        dA = Gw.conj().T @ Gw
        dA = 0.5 * (dA + dA.conj().T)
        stats.A = stats.A + dA
        stats.A = 0.5 * (stats.A + stats.A.conj().T)
    stats.b = stats.b + Gw.conj().T @ dw
    if fallback_hook is not None:
        inc, conv = fallback_hook(Gw)
        iters = 0
    elif literal_power:
        dA = Gw.conj().T @ Gw
        inc, conv = hermitian_top_eigenvalue(0.5 * (dA + dA.conj().T))
        iters = -1
    else:
        inc, conv, iters, _ = top_eigenvalue_nr(Gw, stats.v0())
    stats.last_power = (inc, conv, iters)
    if not conv:
        K = Gw @ Gw.conj().T
        inc = float(np.linalg.norm(K, "fro"))  # |dA|_F = |Gw Gw^H|_F
        stats.fallbacks += 1
    stats.L = stats.L + max(inc, 0.0)
    stats.pulse_count += 1
    return stats


def online_fista_pulse(stats, c_hat, momentum_t, lam, steps, reset_momentum=False):
    if stats.pulse_count < 1:
        raise RuntimeError("no pulses accumulated yet")
    tau = 1.0 / stats.L
    t0 = 1.0 if reset_momentum else float(momentum_t)
    return fista_loop(stats.matvec, np.ascontiguousarray(stats.b.real),
                      np.ascontiguousarray(c_hat, dtype=np.float64), t0, tau, lam * tau, int(steps))


def reconstruct(ell_idx, ell_w, n, c):
    out = np.zeros(n)
    j, l = np.nonzero(ell_idx >= 0)
    np.add.at(out, ell_idx[j, l], ell_w[j, l] * np.asarray(c)[j])
    return out


def run_workload(omega, positions, d, sigma2, ell_idx, ell_w, xyz, steps, lam_rel,
                 n_pulses=None, trace=False):
    """The streaming loop of harness.py:282-287 on a geometric workload, with the
    lambda_n = lam_rel * max|b_n| rule."""
    m = ell_idx.shape[0]
    stats = OracleStats(m)
    c = np.zeros(m)
    t = 1.0
    n_pulses = positions.shape[0] if n_pulses is None else n_pulses
    hist = {"L": [], "lam": [], "c": [], "t": [], "iters": []}
    for k in range(n_pulses):
        F = forward_matrix(omega, positions[k], xyz)
        G = compose_ell(F, ell_idx, ell_w)
        accumulate(stats, G, d[k], sigma2)
        lam = lam_rel * float(np.abs(stats.b).max())
        c, t = online_fista_pulse(stats, c, t, lam, steps)
        hist["L"].append(stats.L)
        hist["lam"].append(lam)
        hist["t"].append(t)
        hist["iters"].append(stats.last_power[2])
        if trace:
            hist["c"].append(c.copy())
    return stats, c, t, hist
