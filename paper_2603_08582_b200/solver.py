"""Reference-shaped streaming solver API over the device engine.

Mirrors solver.py:19-240 of the reference: ``NoiseCovariance``,
``PulseMeasurement``, ``SufficientStatistics``, ``SolverState``,
``SolverConfig``, ``accumulate``, ``online_fista_pulse``,
``hermitian_top_eigenvalue``, ``soft_threshold``, ``reconstruct``.

Semantics versus the reference:
  * ``accumulate`` moves the statistics: the device state is updated in place
    and a fresh ``SufficientStatistics`` view is returned; the view passed in
    becomes stale and raises if read (every reference caller rebinds
    linearly, harness.py:284-287).
  * ``online_fista_pulse`` keeps value semantics on (c_hat, t): it reads c0
    and t0 from the state it is given and returns a new state with a new
    coefficient buffer that shares the statistics (solver.py:226).
  * Dense-pulse (atom-space) statistics up to EXACT_MAX_ATOMS atoms keep the
    complex A in fp64 on the device exactly as the reference does
    (``keep_complex``): ``stats.A``, the reference's dataclass constructor
    ``SufficientStatistics(A=..., b=..., L=...)`` and its hex-text checkpoint
    work unchanged; FISTA reads fp32 Re(A) tiles derived from it.  Larger
    statistics keep only Re(A) (the loop never reads Im(A), solver.py:214-222):
    ``stats.A_re`` materialises it and ``stats.A`` raises.
  * Statistics fed by geometric pulses live in pixel space: G = F H with a
    static H gives A = H^T B H and b = H^T beta (B = sum F^H F / sigma^2), so
    the engine keeps Re(B) (N x N) and beta; ``A_re`` and ``b`` are derived on
    request.  Dense pulses (explicit G) keep atom-space statistics.
  * ``SolverConfig`` accepts ``lam_rel`` (lambda = lam_rel * max|b|, evaluated
    on the device after the pulse) as an extension.
"""

import math
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, ptr
from .dictionary import EdgeletDictionary, synthesize
from .engine import Engine
from .geometry import PulseGeometry, SceneGrid, pixel_positions

DEFAULT_PRECISION = "auto"  # engine.AUTO_DIRICHLET_MIN_NFREQ
# atom-space statistics up to this many atoms keep the complex A (M^2 complex128
# on the device: 268 MB at 4096)
EXACT_MAX_ATOMS = 4096


class NoiseCovariance:
    """R = sigma^2 I or a full Hermitian positive-definite matrix (solver.py:19-68).

    Matrix covariances are handled by whitening the pulse on the host
    (G~ = R^-1/2 G, d~ = R^-1/2 d, an N_r x N_r product) before the device
    update, which then sees sigma^2 = 1.
    """

    def __init__(self, sigma2=None, matrix=None):
        if (sigma2 is None) == (matrix is None):
            raise ValueError("give exactly one of sigma2 or matrix")
        if matrix is None:
            self.sigma2 = float(sigma2)
            if not self.sigma2 > 0.0:
                raise ValueError("sigma2 must be positive")
            self.matrix = None
            self._inv = None
            self._inv_sqrt = None
        else:
            R = np.asarray(matrix, dtype=np.complex128)
            if R.ndim != 2 or R.shape[0] != R.shape[1]:
                raise ValueError("covariance matrix must be square")
            if not np.allclose(R, R.conj().T, rtol=1e-12, atol=1e-12):
                raise ValueError("covariance matrix must be Hermitian")
            try:
                np.linalg.cholesky(R)
            except np.linalg.LinAlgError:
                raise ValueError("covariance matrix must be positive definite") from None
            w, U = np.linalg.eigh(R)
            self.sigma2 = None
            self.matrix = R
            self._inv = (U / w) @ U.conj().T
            self._inv_sqrt = (U / np.sqrt(w)) @ U.conj().T

    @classmethod
    def from_sigma(cls, sigma):
        """Scalar noise level; sigma = 0 is the noiseless convention R = I (solver.py:52-58)."""
        s = float(sigma)
        if s < 0.0:
            raise ValueError("sigma must be nonnegative")
        return cls(sigma2=s * s if s > 0.0 else 1.0)

    def apply_inverse(self, x):
        if self.matrix is None:
            return x / self.sigma2
        return self._inv @ x

    def apply_inverse_sqrt(self, x):
        if self.matrix is None:
            return x / math.sqrt(self.sigma2)
        return self._inv_sqrt @ x


@dataclass
class PulseMeasurement:
    """One pulse's data d, explicit operator G, and noise covariance (solver.py:71-85)."""

    d: np.ndarray
    G: np.ndarray
    noise_cov: NoiseCovariance

    def __post_init__(self):
        self.d = np.asarray(self.d, dtype=np.complex128)
        self.G = np.asarray(self.G, dtype=np.complex128)
        if self.d.ndim != 1 or self.G.ndim != 2 or self.G.shape[0] != self.d.shape[0]:
            raise ValueError("measurement dimensions are inconsistent")
        if self.noise_cov.matrix is not None and self.noise_cov.matrix.shape[0] != self.d.shape[0]:
            raise ValueError("noise covariance does not match the data length")

    @property
    def n_atoms(self):
        return self.G.shape[1]


@dataclass
class GeometricPulse:
    """A pulse described by geometry: the engine synthesises F and G = F H itself.

    ``geometry`` is a PulseGeometry (platform position + angular frequencies),
    ``d`` the N_r complex samples, ``noise_cov`` scalar only.  ``grid`` and
    ``dictionary`` bind the pulse to a scene; ``.G`` materialises the dense
    operator (for tests and oracles only).
    """

    d: np.ndarray
    geometry: PulseGeometry
    noise_cov: NoiseCovariance
    grid: SceneGrid = None
    dictionary: EdgeletDictionary = None

    def __post_init__(self):
        self.d = np.asarray(self.d, dtype=np.complex128)
        if self.d.ndim != 1 or self.d.shape[0] != self.geometry.frequencies.shape[0]:
            raise ValueError("measurement dimensions are inconsistent")
        if self.noise_cov.matrix is not None:
            raise ValueError("geometric pulses take a scalar noise covariance")

    @property
    def n_atoms(self):
        return self.dictionary.m_atoms

    @property
    def G(self):
        from .dictionary import compose
        from .geometry import build_forward_matrix

        return compose(build_forward_matrix(self.geometry, self.grid), self.dictionary)


class SufficientStatistics:
    """Device-resident (A, b, L, pulse_count, fallbacks) (solver.py:88-109).

    Two constructors: ``SufficientStatistics(m_atoms, l_floor, ...)`` (engine
    options as keywords) and the reference dataclass form
    ``SufficientStatistics(A, b, L, pulse_count=0, power_iteration_fallbacks=0)``
    (positional or keyword), which uploads given complex statistics into a
    keep_complex atom-space engine."""

    def __init__(self, m_atoms=None, l_floor=1e-12, precision=DEFAULT_PRECISION, device=0,
                 n_freq=None, dictionary=None, grid=None, mode=None, keep_complex=None, *,
                 A=None, b=None, L=None, pulse_count=0, power_iteration_fallbacks=0):
        if isinstance(m_atoms, np.ndarray) or A is not None:
            if A is None:  # positional reference form (A, b, L, pulse_count, fallbacks)
                A, b, L = m_atoms, l_floor, precision
                pulse_count = device if isinstance(device, (int, np.integer)) and device else pulse_count
                power_iteration_fallbacks = n_freq or power_iteration_fallbacks
                precision, device, n_freq = DEFAULT_PRECISION, 0, None
            self._init_from_fields(A, b, L, pulse_count, power_iteration_fallbacks)
            return
        m = int(m_atoms)
        if m < 1:
            raise ValueError("need at least one atom")
        if not l_floor > 0.0:
            raise ValueError("l_floor must be positive")
        self.m_atoms = m
        self.l_floor = float(l_floor)
        self.precision = precision
        self.device = device
        self._dictionary = dictionary
        self._grid = grid
        self._engine = None
        self._version = 0
        self._mode = mode
        self._keep_complex = keep_complex
        if n_freq is not None:
            self._make_engine(int(n_freq))

    def _init_from_fields(self, A, b, L, pulse_count, fallbacks):
        A = np.asarray(A, dtype=np.complex128)
        b = np.asarray(b, dtype=np.complex128)
        if A.ndim != 2 or A.shape[0] != A.shape[1] or b.shape != (A.shape[0],):
            raise ValueError("statistics dimensions are inconsistent")
        self.m_atoms = A.shape[0]
        self.l_floor = 1e-12
        self.precision = DEFAULT_PRECISION
        self.device = 0
        self._dictionary = self._grid = None
        self._engine = None
        self._version = 0
        self._mode = "atom"
        self._keep_complex = True
        self._dense = True
        self._make_engine(1)
        self._engine.set_stats_complex(A, b, float(L), int(pulse_count), int(fallbacks))
        self._version = self._engine.version

    @classmethod
    def empty(cls, m_atoms, l_floor=1e-12, **kw):
        return cls(m_atoms, l_floor, **kw)

    # -- engine management ---------------------------------------------------
    def _make_engine(self, n_freq, carry=None):
        ell_idx = ell_w = xyz = None
        if self._dictionary is not None:
            ell_idx, ell_w = self._dictionary.ell_idx, self._dictionary.ell_w
            if self._grid is not None:
                xyz = pixel_positions(self._grid)
        keep = self._keep_complex
        if keep is None:  # dense pulses at the reference-API scale: keep the complex A exactly
            keep = getattr(self, "_dense", False) and self.m_atoms <= EXACT_MAX_ATOMS
        self._engine = Engine(self.m_atoms, n_freq, ell_idx, ell_w, xyz, self.precision,
                              self.l_floor, self.device, mode=self._mode, keep_complex=keep)
        if carry is not None:
            if self._engine.mode == "pixel":
                self._engine.set_pixel_stats(*carry)
            elif self._engine.keep_complex:
                self._engine.set_stats_complex(*carry)
            else:
                self._engine.set_stats(*carry)
        self._version = self._engine.version

    def _engine_for(self, n_freq):
        if self._engine is None:
            self._make_engine(max(int(n_freq), 1))
        elif n_freq > self._engine.n_freq:
            # grow the per-pulse capacity; carry the statistics over
            L, n, fb, _ = self._engine.scalars()
            if self._engine.mode == "pixel":
                carry = (*self._engine.get_pixel_stats(), L, n, fb)
            elif self._engine.keep_complex:
                carry = (self._engine.get_A(), self._engine.get_b(), L, n, fb)
            else:
                carry = (self._engine.get_A_re(), self._engine.get_b(), L, n, fb)
            self._engine.close()
            self._make_engine(int(n_freq), carry)
        return self._engine

    def _check_live(self):
        if self._engine is not None and self._version != self._engine.version:
            raise RuntimeError(
                "these statistics were advanced by a later accumulate(); use the returned object")

    def _view(self):
        new = SufficientStatistics.__new__(SufficientStatistics)
        new.__dict__.update(self.__dict__)
        new._version = self._engine.version
        return new

    # -- reference fields --------------------------------------------------------
    @property
    def engine(self):
        self._check_live()
        return self._engine

    @property
    def L(self):
        self._check_live()
        if self._engine is None:
            return self.l_floor
        return self._engine.scalars()[0]

    @property
    def pulse_count(self):
        self._check_live()
        return 0 if self._engine is None else self._engine.scalars()[1]

    @property
    def power_iteration_fallbacks(self):
        self._check_live()
        return 0 if self._engine is None else self._engine.scalars()[2]

    @property
    def b(self):
        self._check_live()
        if self._engine is None:
            return np.zeros(self.m_atoms, dtype=np.complex128)
        return self._engine.get_b()

    @property
    def A_re(self):
        """Re(A) as a dense symmetric float64 matrix."""
        self._check_live()
        if self._engine is None:
            return np.zeros((self.m_atoms, self.m_atoms))
        if self._engine.keep_complex:
            return np.ascontiguousarray(self._engine.get_A().real)
        return self._engine.get_A_re()

    @property
    def A(self):
        """The complex A (keep_complex statistics; zeros before the first pulse)."""
        self._check_live()
        if self._engine is None:
            return np.zeros((self.m_atoms, self.m_atoms), dtype=np.complex128)
        if not self._engine.keep_complex:
            raise AttributeError(
                "these statistics keep only Re(A) on the device (pixel space, or more than "
                f"{EXACT_MAX_ATOMS} atoms; the solver never reads Im(A)); use .A_re")
        return self._engine.get_A()


class _PinnedPool:
    """Page-locked float64 host buffers recycled when the numpy view handed out
    over them is garbage-collected (value semantics: a buffer is never reused
    while a caller can still see it)."""

    RESERVE = 8  # buffers page-locked at a size's first use (results in flight + slack)

    def __init__(self):
        self._free = {}

    def get(self, n):
        import torch

        lst = self._free.get(n)
        if lst is None:
            # page-locking is slow (a driver call per buffer): pay it once, at the
            # first result of this size, not along the stream
            lst = self._free[n] = [torch.empty(n, dtype=torch.float64, pin_memory=True)
                                   for _ in range(self.RESERVE)]
        if lst:
            return lst.pop()
        return torch.empty(n, dtype=torch.float64, pin_memory=True)

    def put(self, t):
        self._free.setdefault(t.numel(), []).append(t)


_PINNED = _PinnedPool()
_WARMED = set()  # (device, m_atoms) whose result buffers the allocator has reserved
_COPY_STREAMS = {}


def _copy_stream(dev):
    import torch

    s = _COPY_STREAMS.get(dev)
    if s is None:
        s = _COPY_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return s


class SolverState:
    """(c_hat, momentum_t, stats) with a device-resident coefficient vector (solver.py:112-120).

    ``online_fista_pulse`` starts the device->host copy of c_hat into page-locked
    memory as soon as the FISTA launch is queued; reading ``c_hat`` waits for
    that copy only, so a caller that reads pulse k's result after queueing pulse
    k+1 keeps the device busy (the copy overlaps the next pulse's work)."""

    # read-only host views handed out by c_hat -> their device buffer, so a
    # state rebuilt from ``old.c_hat`` (harness.py:286) needs no re-upload
    _device_of = {}

    def __init__(self, c_hat, momentum_t, stats):
        self.momentum_t = float(momentum_t)
        self.stats = stats
        self._c_host = None
        self._c_dev = None
        self._pending = None
        if hasattr(c_hat, "data_ptr"):
            self._c_dev = c_hat
        else:
            arr = np.asarray(c_hat, dtype=np.float64)
            entry = SolverState._device_of.get(id(arr))
            if entry is not None and entry[0]() is arr:
                self._c_dev = entry[1]
            self._c_host = arr

    @classmethod
    def initial(cls, m_atoms, l_floor=1e-12, **kw):
        return cls(np.zeros(int(m_atoms)), 1.0, SufficientStatistics.empty(m_atoms, l_floor, **kw))

    def _start_host_copy(self):
        # on a side copy stream ordered after the FISTA output, so the caller's
        # stream (and the next pulse's FISTA, joined to it) never waits on PCIe
        import torch

        dev = self._c_dev.device
        buf = _PINNED.get(self._c_dev.numel())
        cs = _copy_stream(dev)
        cs.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(cs):
            buf.copy_(self._c_dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        self._c_dev.record_stream(cs)  # not recycled before the copy has read it
        self._pending = (buf, ev)

    @property
    def c_hat(self):
        if self._c_host is None:
            if self._pending is not None:
                buf, ev = self._pending
                self._pending = None
                ev.synchronize()
                arr = buf.numpy()
                weakref.finalize(arr, _PINNED.put, buf)
            else:
                arr = self._c_dev.cpu().numpy()
            arr.flags.writeable = False
            self._c_host = arr
            key = id(arr)
            SolverState._device_of[key] = (weakref.ref(arr), self._c_dev)
            weakref.finalize(arr, SolverState._device_of.pop, key, None)
        return self._c_host

    @c_hat.setter
    def c_hat(self, value):
        self._c_host = np.asarray(value, dtype=np.float64)
        self._c_dev = None
        self._pending = None

    def c_device(self, device):
        import torch

        if self._c_dev is None:
            self._c_dev = torch.from_numpy(np.ascontiguousarray(self._c_host, dtype=np.float64)).to(
                f"cuda:{device}")
        return self._c_dev


@dataclass
class SolverConfig:
    """FISTA settings (solver.py:123-136); ``lam_rel`` is the device-side lambda rule."""

    lam: float = None
    inner_steps: int = 20
    l_floor: float = 1e-12
    reset_momentum: bool = False
    lam_rel: float = 0.0

    def __post_init__(self):
        if self.lam is None:
            if not self.lam_rel > 0.0:
                raise ValueError("lambda must be positive")
        elif not self.lam > 0.0:
            raise ValueError("lambda must be positive")
        if int(self.inner_steps) < 1:
            raise ValueError("inner_steps must be at least 1")
        if not self.l_floor > 0.0:
            raise ValueError("l_floor must be positive")


def accumulate(stats, pulse):
    """Fold one pulse into (A, b, L) on the device (solver.py:186-206)."""
    stats._check_live()
    if pulse.n_atoms != stats.m_atoms:
        raise ValueError("pulse operator does not match the atom count")
    if isinstance(pulse, GeometricPulse):
        if stats._dictionary is None:
            stats._dictionary, stats._grid = pulse.dictionary, pulse.grid
        eng = stats._engine_for(pulse.d.shape[0])
        if eng.n_freq != pulse.d.shape[0]:
            raise ValueError("geometric pulses must keep the engine's n_freq")
        eng.accumulate_geom(pulse.geometry.position, pulse.geometry.frequencies, pulse.d,
                            pulse.noise_cov.sigma2)
    else:
        if stats._engine is not None and stats._engine.mode == "pixel":
            raise RuntimeError("pixel-space statistics accept geometric pulses only")
        if stats._engine is None:
            stats._mode = "atom"
            stats._dense = True
        cov = pulse.noise_cov
        if cov.matrix is None:
            G, d, s2 = pulse.G, pulse.d, cov.sigma2
        else:  # whiten: G^H R^-1 G = (R^-1/2 G)^H (R^-1/2 G)
            G, d, s2 = cov.apply_inverse_sqrt(pulse.G), cov.apply_inverse_sqrt(pulse.d), 1.0
        eng = stats._engine_for(pulse.d.shape[0])
        hook = _power_hook()
        if hook is not None and eng.keep_complex:
            _accumulate_with_hook(eng, G, d, s2, hook)
        else:
            eng.accumulate_dense(G, d, s2)
    return stats._view()


def _power_hook():
    """The module's hermitian_top_eigenvalue when a caller replaced it (the
    reference's fault-injection seam, test_solver.py:157-167), else None."""
    f = globals().get("hermitian_top_eigenvalue")
    return None if f is _DEVICE_TOP_EIGENVALUE else f


def _accumulate_with_hook(eng, G, d, s2, hook):
    """accumulate() with a caller-supplied top-eigenvalue routine: the engine
    folds the pulse into A and b, then L gets the hook's increment on the
    symmetrised dA, or the Frobenius fallback (solver.py:194-199)."""
    A0 = eng.get_A()
    L0, n0, fb0, _ = eng.scalars()
    eng.accumulate_dense(G, d, s2)
    dA = eng.get_A() - A0
    dA = 0.5 * (dA + dA.conj().T)
    inc, converged = hook(dA)
    fb = fb0
    if not converged:
        inc = float(np.linalg.norm(dA, "fro"))
        fb += 1
    eng.set_scalars(L0 + max(float(inc), 0.0), n0 + 1, fb)


def online_fista_pulse(state, cfg):
    """cfg.inner_steps warm-started FISTA steps on the device (solver.py:209-226)."""
    import torch

    stats = state.stats
    stats._check_live()
    if stats._engine is None:
        raise RuntimeError("no pulses accumulated yet")  # the engine re-checks its own count
    eng = stats._engine
    c0 = state.c_device(eng.device)
    key = (c0.device, stats.m_atoms)
    if key not in _WARMED:
        # results live on the device until their host copies are read; have the
        # caching allocator reserve a dozen result buffers now (one driver
        # allocation here) rather than grow along the stream
        _WARMED.add(key)
        del [torch.empty(stats.m_atoms, dtype=torch.float64, device=c0.device) for _ in range(12)][:]
    c_out = torch.empty(stats.m_atoms, dtype=torch.float64, device=c0.device)
    t0 = 1.0 if cfg.reset_momentum else float(state.momentum_t)
    lam = float(cfg.lam) if cfg.lam is not None else 0.0
    t = eng.fista(c0, c_out, int(cfg.inner_steps), t0, lam=lam, lam_rel=float(cfg.lam_rel))
    out = SolverState(c_out, t, stats)
    out._start_host_copy()
    return out


def batch_fista(pulses, cfg, iterations):
    """Classical FISTA on the full pulse set from a zero start (solver.py:267-291).

    The device batch oracle: every pulse is folded into fresh pixel-space
    statistics, L = lambda_max(sum_k G_k^H G_k / sigma_k^2) comes from the
    reference's power iteration run matrix-free on the device, floored at
    ``cfg.l_floor``, and ``iterations`` FISTA steps run from c = 0, t = 1 with
    lambda = ``cfg.lam`` (or ``cfg.lam_rel`` max|b|).  If that power iteration
    does not converge, the reference's Frobenius fallback runs on the exact
    complex A of the retained pulses (up to EXACT_MAX_ATOMS atoms).
    """
    if int(iterations) < 1:
        raise ValueError("iterations must be at least 1")
    if not pulses:
        raise ValueError("need at least one pulse")
    if not all(isinstance(p, GeometricPulse) for p in pulses):
        return _batch_fista_dense(pulses, cfg, iterations)
    p0 = pulses[0]
    m = p0.n_atoms
    stats = SufficientStatistics.empty(m, cfg.l_floor, dictionary=p0.dictionary, grid=p0.grid,
                                       n_freq=p0.d.shape[0])
    for p in pulses:
        stats = accumulate(stats, p)
    eng = stats.engine
    if eng.mode != "pixel":
        raise ValueError("the device batch oracle needs pixel-space statistics")
    gam = np.stack([np.asarray(p.geometry.position, dtype=np.float64) for p in pulses])
    lam_max, converged = eng.batch_lipschitz(gam, p0.geometry.frequencies,
                                             [p.noise_cov.sigma2 for p in pulses])
    if not converged:
        # the reference's Frobenius fallback (solver.py:281-283) needs |A|_F of the
        # full batch matrix: rebuild the exact atom-space statistics of the
        # retained pulses on the device (their operators composed there) and take
        # the dense path, as long as the complex A fits
        if m > EXACT_MAX_ATOMS:
            raise RuntimeError("batch power iteration did not converge and the Frobenius "
                               f"fallback needs the dense A (at most {EXACT_MAX_ATOMS} atoms)")
        return _batch_fista_dense([PulseMeasurement(p.d, p.G, p.noise_cov) for p in pulses],
                                  cfg, iterations)
    L = max(lam_max, cfg.l_floor)
    _, n, fb, _ = eng.scalars()
    eng.set_pixel_stats(None, None, L, n, fb)
    c = np.empty(m)
    lam = float(cfg.lam) if cfg.lam is not None else 0.0
    eng.fista(np.zeros(m), c, int(iterations), 1.0, lam=lam, lam_rel=float(cfg.lam_rel))
    return c


def _batch_fista_dense(pulses, cfg, iterations):
    """Dense pulses: exact atom-space statistics of all pulses, L from the
    reference's power iteration on the full A (device, M space; Frobenius
    fallback), floored at l_floor, then ``iterations`` FISTA steps from zero."""
    m = pulses[0].n_atoms
    if m > EXACT_MAX_ATOMS:
        raise ValueError(f"the dense batch oracle keeps the complex A: at most "
                         f"{EXACT_MAX_ATOMS} atoms")
    stats = SufficientStatistics.empty(m, cfg.l_floor, keep_complex=True)
    for p in pulses:
        stats = accumulate(stats, p)
    eng = stats.engine
    A = eng.get_A()
    L, converged = hermitian_top_eigenvalue(A)
    if not converged:
        L = float(np.linalg.norm(A, "fro"))
    L = max(L, cfg.l_floor)
    _, n, fb, _ = eng.scalars()
    eng.set_scalars(L, n, fb)
    c = np.empty(m)
    lam = float(cfg.lam) if cfg.lam is not None else 0.0
    eng.fista(np.zeros(m), c, int(iterations), 1.0, lam=lam, lam_rel=float(cfg.lam_rel))
    return c


def _whitened(p):
    cov = p.noise_cov
    if cov.matrix is None:
        return p.G, p.d, cov.sigma2
    return cov.apply_inverse_sqrt(p.G), cov.apply_inverse_sqrt(p.d), 1.0


def _residual_terms(c, pulses):
    """(sum_k |d_k - G_k c|^2_{R_k^-1}, Re sum_k G_k^H R_k^-1 (G_k c - d_k)) on the device."""
    import ctypes

    c = np.ascontiguousarray(c, dtype=np.float64)
    if not pulses:
        raise ValueError("need at least one pulse")
    m = pulses[0].n_atoms
    if c.shape != (m,):
        raise ValueError("coefficient vector does not match the atom count")
    grad = np.zeros(m)
    quad = 0.0
    lib = _lib.load()
    for p in pulses:
        G, d, s2 = _whitened(p)
        G = np.ascontiguousarray(G, dtype=np.complex128)
        d = np.ascontiguousarray(d, dtype=np.complex128)
        if G.shape[1] != m:
            raise ValueError("pulse operator does not match the atom count")
        q = ctypes.c_double()
        check(lib.sf_dense_residual(0, ptr(G), ptr(d), G.shape[0], m, ptr(c), float(s2),
                                    ctypes.byref(q), ptr(grad)))
        quad += q.value
    return quad, grad


def batch_objective(c, pulses, lam):
    """Weighted LASSO value over retained pulses (solver.py:243-252), residuals on the device."""
    quad, _ = _residual_terms(c, pulses)
    return 0.5 * quad + lam * float(np.abs(np.asarray(c, dtype=np.float64)).sum())


def batch_gradient(c, pulses):
    """Gradient of the smooth term for real c (solver.py:255-264), on the device."""
    return _residual_terms(c, pulses)[1]


def save_checkpoint(path, state):
    """solver.py:302-332; see checkpoint.save_checkpoint."""
    from .checkpoint import save_checkpoint as _save

    return _save(path, state)


def load_checkpoint(path, *args, **kw):
    """solver.py:335-369; see checkpoint.load_checkpoint."""
    from .checkpoint import load_checkpoint as _load

    return _load(path, *args, **kw)


def hermitian_top_eigenvalue(X, rel_tol=1e-6, max_iter=500):
    """Power iteration with the reference's stopping rule and bias (solver.py:139-175)."""
    import ctypes

    X = np.ascontiguousarray(X, dtype=np.complex128)
    if X.ndim != 2 or X.shape[0] != X.shape[1]:
        raise ValueError("matrix must be square")
    lam = ctypes.c_double()
    conv = ctypes.c_int32()
    check(_lib.load().sf_hermitian_top_eigenvalue(0, ptr(X), X.shape[0], float(rel_tol),
                                                  int(max_iter), ctypes.byref(lam),
                                                  ctypes.byref(conv)))
    return lam.value, bool(conv.value)


_DEVICE_TOP_EIGENVALUE = hermitian_top_eigenvalue


def soft_threshold(u, alpha):
    """Sign/phase-preserving shrinkage u (1 - alpha/|u|)_+ (solver.py:229-240)."""
    if alpha < 0.0:
        raise ValueError("alpha must be nonnegative")
    arr = np.asarray(u)
    is_c = np.iscomplexobj(arr)
    src = np.ascontiguousarray(arr, dtype=np.complex128 if is_c else np.float64)
    out = np.empty_like(src)
    check(_lib.load().sf_soft_threshold(0, ptr(src), src.size, 1 if is_c else 0, float(alpha),
                                        ptr(out)))
    if arr.ndim == 0:
        return out.reshape(()).item()
    return out.reshape(arr.shape)


def reconstruct(state, dictionary):
    """Image synthesis H c on the device (solver.py:294-299)."""
    m = dictionary.m_atoms if hasattr(dictionary, "m_atoms") else np.asarray(dictionary).shape[1]
    c = state.c_hat
    if m != c.shape[0]:
        raise ValueError("dictionary does not match the coefficient vector")
    eng = getattr(state.stats, "_engine", None)
    if (eng is not None and dictionary is state.stats._dictionary and eng.n_pixels > 0):
        return eng.reconstruct(c)
    return synthesize(dictionary, c)
