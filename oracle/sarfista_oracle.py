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


# --- symmetric store: upper-triangle row panels, dgemm / dgemv -------------------------
# OpenBLAS 0.3.30 as shipped with scipy/numpy here returns wrong entries from a
# multithreaded dsyrk at n = 36864 (and numpy's syrk path for P.T @ P segfaults
# there), so the rank update and the symmetric matvec are written with plain
# dgemm / dgemv (numpy's ILP64 BLAS) over row panels of the upper triangle,
# checked against direct dot products in tests/test_oracle.py.
class SymStore:
    """Symmetric n x n matrix held as its upper triangle in C-ordered row panels:
    panel k = rows [k*p, k*p + p) x columns [k*p, n).  The strict lower part of
    each panel's diagonal block is kept at zero."""

    def __init__(self, n, panel=256):
        self.n = int(n)
        self.panel = int(panel)
        self.rows = [np.zeros((min(self.n, i0 + self.panel) - i0, self.n - i0))
                     for i0 in range(0, self.n, self.panel)]

    def rank_update(self, PT):
        """S += P^T P with P = PT.T (k x n)."""
        for k, R in enumerate(self.rows):
            i0 = k * self.panel
            bs = R.shape[0]
            R += PT[i0:i0 + bs] @ PT[i0:].T
            R[:, :bs] = np.triu(R[:, :bs])

    def matvec(self, z):
        y = np.zeros(self.n)
        for k, R in enumerate(self.rows):
            i0 = k * self.panel
            bs = R.shape[0]
            y[i0:i0 + bs] += R @ z[i0:]
            y[i0:] += R.T @ z[i0:i0 + bs]
        return y - self.diagonal() * z

    def diagonal(self):
        return np.concatenate([np.diagonal(R[:, :R.shape[0]]) for R in self.rows])

    def dense(self):
        S = np.zeros((self.n, self.n))
        for k, R in enumerate(self.rows):
            i0 = k * self.panel
            S[i0:i0 + R.shape[0], i0:] = R
        return S + np.triu(S, 1).T


# --- solver.py:88-226 -----------------------------------------------------------------
class OracleStats:
    """(Re A, b, L, n, fallbacks); optionally the full complex A for small M.

    Re(A) is held as its upper triangle (SymStore) and updated with
    A += P^T P, P = [Re G~; Im G~]; the FISTA loop reads it with the symmetric
    matvec.  The stored operator is exactly symmetric, so the reference's
    symmetrisations (solver.py:181, 193) are identities here; ``A_re`` returns
    the full symmetric matrix."""

    def __init__(self, m, l_floor=1e-12, keep_complex=False):
        self._Au = SymStore(m)
        self.A = np.zeros((m, m), dtype=np.complex128) if keep_complex else None
        self.b = np.zeros(m, dtype=np.complex128)
        self.L = float(l_floor)
        self.pulse_count = 0
        self.fallbacks = 0
        self.last_power = None
        self._v0 = None

    @property
    def A_re(self):
        return self._Au.dense()

    def matvec(self, z):
        return self._Au.matvec(z)

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
    PT = np.empty((Gw.shape[1], 2 * Gw.shape[0]))
    PT[:, :Gw.shape[0]] = Gw.real.T
    PT[:, Gw.shape[0]:] = Gw.imag.T
    # A_re (upper) += P^T P  (Re(G^H G) = Gr^T Gr + Gi^T Gi)
    stats._Au.rank_update(PT)
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


def top_eigenvalue_k(K, u0, rel_tol=1e-6, max_iter=500):
    """top_eigenvalue_nr with K = Gw Gw^H and u0 = Gw v0 supplied (
    the iterate sequence of solver.py:157-175)."""
    u = np.asarray(u0, dtype=np.complex128)
    lam_prev = None
    delta_prev = None
    it = 0
    for it in range(int(max_iter)):
        lam = float(np.real(np.vdot(u, u)))
        Ku = K @ u
        norm_w = math.sqrt(max(float(np.real(np.vdot(u, Ku))), 0.0))
        if norm_w == 0.0:
            return 0.0, True, it + 1
        u = Ku / norm_w
        if lam_prev is not None:
            delta = lam - lam_prev
            if abs(delta) <= rel_tol * max(abs(lam), 1e-300):
                tail = 0.0
                if delta_prev is not None and abs(delta_prev) > abs(delta) > 0.0:
                    q = delta / delta_prev
                    if 0.0 < q < 1.0:
                        tail = delta * q / (1.0 - q)
                return lam + tail + abs(delta), True, it + 1
            delta_prev = delta
        lam_prev = lam
    return (lam_prev if lam_prev is not None else 0.0), False, it + 1


# --- pixel-space restatement (exact: A = H^T B H, b = H^T beta) ---------------------
def sparse_dictionary(ell_idx, ell_w, n):
    """H (N x M) as scipy CSR from the ELL table."""
    from scipy import sparse

    j, l = np.nonzero(ell_idx >= 0)
    return sparse.csr_matrix((ell_w[j, l], (ell_idx[j, l], j)), shape=(n, ell_idx.shape[0]))


class PixelOracleStats:
    """The same statistics as OracleStats, held in pixel space.

    Every geometric pulse has G = F H with the static dictionary H, so
      Re(A) = H^T Re(B) H,  B = sum_k F_k^H F_k / sigma_k^2   (N x N)
      b     = H^T beta,     beta = sum_k F_k^H d_k / sigma_k^2
    exactly (the association order of solver.py:178-193 changes, nothing else).
    Re(B) is the upper triangle of a SymStore updated with
    P = [Re F~; Im F~] (Re(F^H F) = Fr^T Fr + Fi^T Fi), as
    OracleStats does for Re(A); the FISTA matvec is Re(A) z = H^T (Re(B) (H z)).
    The Lipschitz increment runs the N_r-space power iteration on
    K = G~ G~^H = F~ (H H^T) F~^H from u0 = F~ (H v0) -- the iterate sequence of
    solver.py:157-175.  Gated against the M-space OracleStats to
    1e-12 (tests/test_oracle.py, tests/golden/make_config_golden.py)."""

    def __init__(self, ell_idx, ell_w, n, l_floor=1e-12):
        self.H = sparse_dictionary(ell_idx, ell_w, n)
        self.HT = self.H.T.tocsr()
        self.Q = (self.H @ self.HT).tocsr()
        m = ell_idx.shape[0]
        self._Bu = SymStore(n)
        self.beta = np.zeros(n, dtype=np.complex128)
        self.L = float(l_floor)
        self.pulse_count = 0
        self.fallbacks = 0
        self.last_power = None
        self._v0 = counter_unit_complex_vector(m)
        self._hv0 = self.H @ self._v0

    @property
    def b(self):
        return self.HT @ self.beta

    @property
    def B_re(self):
        return self._Bu.dense()

    def matvec(self, z):
        return self.HT @ self._Bu.matvec(self.H @ z)


def accumulate_pixel(stats, F, d, sigma2):
    """accumulate (solver.py:186-206) for a geometric pulse G = F H, scalar R = sigma^2 I."""
    s = 1.0 / math.sqrt(sigma2)
    Fw = np.asarray(F, dtype=np.complex128) * s
    dw = np.asarray(d, dtype=np.complex128) * s
    n_r, n = Fw.shape
    PT = np.empty((n, 2 * n_r))
    PT[:, :n_r] = Fw.real.T
    PT[:, n_r:] = Fw.imag.T
    stats._Bu.rank_update(PT)
    stats.beta = stats.beta + Fw.conj().T @ dw
    K = Fw @ np.asarray(stats.Q @ Fw.conj().T)
    u0 = Fw @ stats._hv0
    inc, conv, iters = top_eigenvalue_k(K, u0)
    stats.last_power = (inc, conv, iters)
    if not conv:
        inc = float(np.linalg.norm(K, "fro"))
        stats.fallbacks += 1
    stats.L = stats.L + max(inc, 0.0)
    stats.pulse_count += 1
    return stats


def run_workload_pixel(omega, positions, d, sigma2, ell_idx, ell_w, xyz, steps, lam_rel,
                       n_pulses=None, trace_at=(), on_pulse=None):
    """run_workload (the streaming loop of harness.py:282-287 with the lambda rule)
    on the pixel-space statistics.  ``trace_at``: pulse indices whose c is kept."""
    n = xyz.shape[0]
    stats = PixelOracleStats(ell_idx, ell_w, n)
    m = ell_idx.shape[0]
    c = np.zeros(m)
    t = 1.0
    n_pulses = positions.shape[0] if n_pulses is None else n_pulses
    trace_at = set(int(k) for k in trace_at)
    hist = {"L": [], "lam": [], "c": {}, "t": [], "iters": [], "conv": []}
    for k in range(n_pulses):
        F = forward_matrix(omega, positions[k], xyz)
        accumulate_pixel(stats, F, d[k], sigma2)
        b = stats.b
        lam = lam_rel * float(np.abs(b).max())
        if stats.pulse_count < 1:
            raise RuntimeError("no pulses accumulated yet")
        tau = 1.0 / stats.L
        c, t = fista_loop(stats.matvec, np.ascontiguousarray(b.real), c, t, tau, lam * tau,
                          int(steps))
        hist["L"].append(stats.L)
        hist["lam"].append(lam)
        hist["t"].append(t)
        hist["iters"].append(stats.last_power[2])
        hist["conv"].append(stats.last_power[1])
        if k in trace_at:
            hist["c"][k] = c.copy()
        if on_pulse is not None:
            on_pulse(k, stats, c, t)
    return stats, c, t, hist


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
