"""Handle-level wrapper of the device engine (one ``sf_engine`` per statistics set).

This is the thin layer the reference-shaped API in :mod:`.solver` sits on and
the object ``bench.py`` drives directly.  Device buffers handed to the engine
are torch tensors (plumbing only); the engine itself allocates its state with
cudaMalloc and runs every kernel from ``libsarfista_b200.so``.
"""

import ctypes

import numpy as np

from . import _lib
from ._lib import SF_MEM_DEVICE, SF_MEM_HOST, check, ptr

# precision="auto": closed-form (dirichlet) pixel Gram from this many frequencies
# per pulse up.  Measured on B200 with the state stream at low priority, f16x3 ->
# dirichlet pulses/s: cfg0 (N_r = 64) 9 187 -> 9 260, cfg1 (128) 5 355 -> 5 420
# (flushed) / 6 245 -> 6 358 (warm), cfg2 (64) 111.6k -> 112.9k, cfg3 (256) 504
# -> 546, cfg4 (512) 43.6 -> 71.6: the closed form is the faster (and more
# accurate) pixel Gram at every BASELINE size.
AUTO_DIRICHLET_MIN_NFREQ = 1


def _torch():
    import torch

    return torch


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Engine:
    """Device-resident sufficient statistics (packed symmetric Re(A), b, L, counters).

    Parameters
    ----------
    m_atoms, n_freq : problem sizes (n_freq is the per-pulse capacity, <= 512).
    ell_idx, ell_w  : optional dictionary as an ELL table ``[m_atoms][width]``
                      (index -1 marks an unused slot); required for geometric
                      pulses and for :meth:`reconstruct`.
    pixel_xyz       : ``[n_pixels][3]`` pixel centres (scene.py:93-105).
    precision       : Gram-update arithmetic: "auto" (default), "f16x3", "tf32x3", "tf32",
                      "fp32", or "dirichlet" (pixel mode; the sum over a uniformly spaced
                      frequency grid in closed form, O(1) per stored entry).  "auto" picks
                      "dirichlet" for pixel mode (measured faster than the f16x3 tensor-core
                      contraction at every BASELINE size; frequencies
                      must then be uniformly spaced, as angular_frequencies makes them --
                      pass "f16x3" for other grids) and "f16x3" in atom mode.
    """

    def __init__(self, m_atoms, n_freq, ell_idx=None, ell_w=None, pixel_xyz=None,
                 precision="auto", l_floor=1e-12, device=0, power_max_iter=0,
                 power_rel_tol=0.0, mode=None, batch=1, keep_complex=False):
        lib = _lib.load()
        self.m_atoms = int(m_atoms)
        self.n_freq = int(n_freq)
        self.device = int(device)
        desc = _lib.SfDesc()
        desc.abi_version = _lib.ABI_VERSION
        desc.device = self.device
        desc.m_atoms = self.m_atoms
        desc.n_freq = self.n_freq
        desc.l_floor = float(l_floor)
        desc.power_max_iter = int(power_max_iter)
        desc.power_rel_tol = float(power_rel_tol)
        self.batch = int(batch)
        desc.batch = self.batch
        if mode is None:  # pixel space whenever the pulses can be geometric
            mode = "pixel" if (ell_idx is not None and pixel_xyz is not None) else "atom"
        if mode not in _lib.MODES:
            raise ValueError(f"unknown mode {mode!r}")
        self.mode = mode
        desc.mode = _lib.MODES[mode]
        if precision == "auto":
            precision = ("dirichlet" if mode == "pixel" and self.n_freq >= AUTO_DIRICHLET_MIN_NFREQ
                         else "f16x3")
        if precision not in _lib.PRECISIONS:
            raise ValueError(f"unknown precision {precision!r}")
        self.precision = precision
        desc.precision = _lib.PRECISIONS[precision]
        self.keep_complex = bool(keep_complex)
        desc.keep_complex = 1 if self.keep_complex else 0
        self._keep = []
        self.n_pixels = 0
        if ell_idx is not None:
            idx = np.ascontiguousarray(ell_idx, dtype=np.int32)
            w = _f64(ell_w)
            if idx.ndim != 2 or idx.shape[0] != self.m_atoms or w.shape != idx.shape:
                raise ValueError("ELL table must be [m_atoms][width] for both index and weight")
            desc.ell_width = idx.shape[1]
            desc.ell_idx = idx.ctypes.data
            desc.ell_w = w.ctypes.data
            self._keep += [idx, w]
            if pixel_xyz is not None:
                xyz = _f64(pixel_xyz)
                if xyz.ndim != 2 or xyz.shape[1] != 3:
                    raise ValueError("pixel_xyz must be [n_pixels][3]")
                desc.pixel_xyz = xyz.ctypes.data
                desc.n_pixels = xyz.shape[0]
                self._keep.append(xyz)
            else:
                desc.n_pixels = int(idx.max()) + 1
            self.n_pixels = int(desc.n_pixels)
        handle = ctypes.c_void_p()
        check(lib.sf_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self._lib = lib
        self._keep = []
        self.version = 0  # bumped by every accumulate (stale-handle detection)
        m_pad = ctypes.c_int64()
        tile = ctypes.c_int32()
        n_tiles = ctypes.c_int64()
        nbytes = ctypes.c_int64()
        check(lib.sf_info(self._h, ctypes.byref(m_pad), ctypes.byref(tile),
                          ctypes.byref(n_tiles), ctypes.byref(nbytes)))
        self.m_pad, self.tile = m_pad.value, tile.value
        self.n_tiles, self.device_bytes = n_tiles.value, nbytes.value
        self._bound_stream = None

    def _bind(self):
        """Order engine work after/before torch work: issue on torch's current stream."""
        torch = _torch()
        s = torch.cuda.current_stream(self.device)
        if s.cuda_stream != self._bound_stream:
            check(self._lib.sf_set_stream(self._h, ctypes.c_void_p(s.cuda_stream)))
            self._bound_stream = s.cuda_stream

    # -- lifetime ------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.sf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard(self, rank, world, unique_id=None):
        """Own only this rank's share of the pixel-space state (see sharding.py)."""
        uid = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
        check(self._lib.sf_shard_init(self._h, int(rank), int(world), uid))
        self.rank, self.world = int(rank), int(world)

    def set_stream(self, stream):
        """Issue all further work on a torch.cuda.Stream."""
        check(self._lib.sf_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))
        self._bound_stream = stream.cuda_stream

    def synchronize(self):
        check(self._lib.sf_synchronize(self._h))

    def reset(self, l_floor=1e-12):
        check(self._lib.sf_reset(self._h, float(l_floor)))
        self.version += 1

    # -- per-pulse update -----------------------------------------------------
    def accumulate_geom(self, gamma, omega, d, sigma2):
        """One geometric pulse.  gamma [3], omega [n_freq] float64 and d [n_freq]
        complex128: all numpy (host) or all torch cuda tensors (device-resident)."""
        if hasattr(d, "data_ptr"):
            self._bind()
            g, w, dd, mem = gamma, omega, d, SF_MEM_DEVICE
            if g.numel() != 3 or w.numel() != self.n_freq or dd.numel() != self.n_freq:
                raise ValueError("omega and d must have n_freq entries")
        else:
            g = _f64(gamma).reshape(3)
            w = _f64(omega)
            dd = _c128(d)
            mem = SF_MEM_HOST
            if w.shape != (self.n_freq,) or dd.shape != (self.n_freq,):
                raise ValueError("omega and d must have n_freq entries")
        check(self._lib.sf_accumulate_geom(self._h, ptr(g), ptr(w), ptr(dd), float(sigma2), mem))
        self.version += 1

    def accumulate_dense(self, G, d, sigma2):
        """G [n_r][m_atoms] complex, d [n_r] complex: numpy (host) or torch cuda."""
        if hasattr(G, "data_ptr"):
            torch = _torch()
            if G.dtype != torch.complex128 or d.dtype != torch.complex128:
                raise ValueError("device G and d must be complex128")
            self._bind()
            Gc, dc, mem = G.contiguous(), d.contiguous(), SF_MEM_DEVICE
        else:
            Gc, dc, mem = _c128(G), _c128(d), SF_MEM_HOST
        if Gc.ndim != 2 or Gc.shape[1] != self.m_atoms or dc.shape != (Gc.shape[0],):
            raise ValueError("pulse operator does not match the atom count")
        check(self._lib.sf_accumulate_dense(self._h, ptr(Gc), ptr(dc), int(Gc.shape[0]),
                                            float(sigma2), mem))
        self.version += 1

    # -- FISTA -------------------------------------------------------------------
    def accumulate_geom_batch(self, gammas, omega, d, sigma2):
        """One pulse for each of the engine's `batch` scenes: gammas [B, 3],
        omega [N_r], d [B, N_r] complex, sigma2 [B] (numpy on the host or
        torch cuda tensors: float64 / complex128)."""
        if self.batch < 2:
            raise RuntimeError("not a batched engine")
        if hasattr(d, "data_ptr"):
            self._bind()
            mem = SF_MEM_DEVICE
            g, w, dd, s2 = gammas, omega, d, sigma2
        else:
            mem = SF_MEM_HOST
            g = _f64(gammas)
            w = _f64(omega)
            dd = np.ascontiguousarray(d, dtype=np.complex128)
            s2 = _f64(sigma2)
            if g.shape != (self.batch, 3) or dd.shape != (self.batch, self.n_freq) or \
                    s2.shape != (self.batch,) or w.shape != (self.n_freq,):
                raise ValueError("batched pulse arrays have the wrong shape")
        check(self._lib.sf_accumulate_geom_batch(self._h, ptr(g), ptr(w), ptr(dd), ptr(s2), mem))
        self.version += 1

    def batch_lipschitz(self, gammas, omega, sigma2, rel_tol=1e-6, max_iter=500):
        """(lambda_max, converged) of A = sum_k G_k^H G_k / sigma_k^2 over the given
        geometric pulses (solver.py:139-175 run matrix-free on the device)."""
        g = _f64(np.atleast_2d(gammas))
        w = _f64(omega)
        s2 = _f64(np.atleast_1d(sigma2))
        if g.shape[1] != 3 or s2.shape[0] != g.shape[0] or w.shape != (self.n_freq,):
            raise ValueError("batch pulse arrays have the wrong shape")
        lam = ctypes.c_double()
        conv = ctypes.c_int32()
        check(self._lib.sf_batch_lipschitz(self._h, ptr(g), ptr(w), ptr(s2), g.shape[0],
                                           float(rel_tol), int(max_iter), ctypes.byref(lam),
                                           ctypes.byref(conv)))
        return lam.value, bool(conv.value)

    def batch_scalars(self):
        """(L [B], pulse_count [B], fallbacks [B]) of a batched engine."""
        L = np.empty(self.batch)
        n = np.empty(self.batch, dtype=np.int64)
        fb = np.empty(self.batch, dtype=np.int64)
        check(self._lib.sf_get_batch_scalars(self._h, ptr(L), ptr(n), ptr(fb)))
        return L, n, fb

    def fista(self, c0, c_out, steps, t0, lam=0.0, lam_rel=0.0):
        """Run ``steps`` FISTA iterations from c0 into c_out; returns the new momentum t.

        c0 / c_out are both numpy float64 (host) or both torch float64 cuda tensors.
        """
        mem = SF_MEM_DEVICE if hasattr(c_out, "data_ptr") else SF_MEM_HOST
        if mem == SF_MEM_DEVICE:
            self._bind()
        t = ctypes.c_double()
        check(self._lib.sf_fista(self._h, ptr(c0), ptr(c_out), mem, float(lam),
                                 float(lam_rel), int(steps), float(t0), ctypes.byref(t)))
        return t.value

    # -- readback ------------------------------------------------------------------
    def scalars(self):
        L = ctypes.c_double()
        n = ctypes.c_int64()
        fb = ctypes.c_int64()
        lam = ctypes.c_double()
        check(self._lib.sf_get_scalars(self._h, ctypes.byref(L), ctypes.byref(n),
                                       ctypes.byref(fb), ctypes.byref(lam)))
        return L.value, n.value, fb.value, lam.value

    def power_diag(self):
        """Last power iteration: (increment, iterations, converged, |dA|_F)."""
        out = np.empty(4)
        check(self._lib.sf_get_power_diag(self._h, ptr(out)))
        return float(out[0]), int(out[1]), bool(out[2]), float(out[3])

    def probe_store_read(self, iters=50):
        """Mean microseconds of a plain streaming read of the current tile store."""
        us = ctypes.c_double()
        check(self._lib.sf_probe_store_read(self._h, int(iters), ctypes.byref(us)))
        return us.value

    def probe_matvec(self, iters=50, dense=False):
        """Mean microseconds of one FISTA matvec launch alone (back to back);
        dense=True reads every tile element (the support-blind ceiling)."""
        us = ctypes.c_double()
        check(self._lib.sf_probe_matvec(self._h, int(iters), int(bool(dense)), ctypes.byref(us)))
        return us.value

    def apply_store(self, x, y, dense=False):
        """y = Re(B) x through the product matvec kernels: x a float32 CUDA tensor
        of n_pad entries, y a float64 CUDA tensor of n_pixels (pixel mode)."""
        check(self._lib.sf_apply_store(self._h, ctypes.c_void_p(x.data_ptr()),
                                       ctypes.c_void_p(y.data_ptr()), int(bool(dense))))

    def get_b(self):
        out = np.empty(self.m_atoms, dtype=np.complex128)
        check(self._lib.sf_get_b(self._h, ptr(out), SF_MEM_HOST))
        return out

    def get_A(self):
        """The complex A [M][M] of a keep_complex engine (stats.A, solver.py:88-109)."""
        out = np.empty((self.m_atoms, self.m_atoms), dtype=np.complex128)
        check(self._lib.sf_get_A(self._h, ptr(out), SF_MEM_HOST))
        return out

    def set_stats_complex(self, A, b, L, pulse_count, fallbacks):
        a = None if A is None else _c128(A)
        bb = None if b is None else _c128(b)
        if a is not None and a.shape != (self.m_atoms, self.m_atoms):
            raise ValueError("A shape mismatch")
        if bb is not None and bb.shape != (self.m_atoms,):
            raise ValueError("b shape mismatch")
        check(self._lib.sf_set_stats_complex(self._h, ptr(a), ptr(bb), float(L), int(pulse_count),
                                             int(fallbacks), SF_MEM_HOST))
        self.version += 1

    def set_scalars(self, L, pulse_count, fallbacks):
        """L and the counters only (A and b unchanged)."""
        check(self._lib.sf_set_stats(self._h, None, None, float(L), int(pulse_count),
                                     int(fallbacks), SF_MEM_HOST))

    def get_A_re(self):
        out = np.empty((self.m_atoms, self.m_atoms), dtype=np.float64)
        check(self._lib.sf_get_A_re(self._h, ptr(out), SF_MEM_HOST))
        return out

    def get_pixel_stats(self):
        """(Re(B) [N][N], beta [N]) of a pixel-space engine."""
        B = np.empty((self.n_pixels, self.n_pixels), dtype=np.float64)
        beta = np.empty(self.n_pixels, dtype=np.complex128)
        check(self._lib.sf_get_pixel_stats(self._h, ptr(B), ptr(beta), SF_MEM_HOST))
        return B, beta

    def n_tiles_local(self):
        """Stored tiles this engine updates and multiplies with (all, unless sharded)."""
        n = ctypes.c_int64()
        check(self._lib.sf_tile_store(self._h, ctypes.byref(n), None, None))
        return n.value

    def get_tiles(self):
        """(tile_ij [n][2] int32, tiles [n][128*128] float32) owned by this rank."""
        n = ctypes.c_int64()
        nt = ctypes.c_int64()
        check(self._lib.sf_tile_store(self._h, ctypes.byref(n), ctypes.byref(nt), None))
        ij = np.empty((n.value, 2), dtype=np.int32)
        check(self._lib.sf_tile_store(self._h, None, None, ptr(ij)))
        tiles = np.empty((n.value, 128 * 128), dtype=np.float32)
        check(self._lib.sf_copy_tiles(self._h, ptr(tiles), 0, SF_MEM_HOST))
        return ij, tiles

    def set_tiles(self, tile_ij, tiles):
        n = ctypes.c_int64()
        check(self._lib.sf_tile_store(self._h, ctypes.byref(n), None, None))
        ij = np.empty((n.value, 2), dtype=np.int32)
        check(self._lib.sf_tile_store(self._h, None, None, ptr(ij)))
        if not np.array_equal(ij, np.asarray(tile_ij)):
            raise ValueError("checkpoint tiles do not match this engine's tile ownership")
        t = np.ascontiguousarray(tiles, dtype=np.float32)
        check(self._lib.sf_copy_tiles(self._h, ptr(t), 1, SF_MEM_HOST))

    def get_bp(self):
        """(image_sum [N] complex = sum_k F_k^H d_k, pulse_count) -- baseline.py:23-33."""
        img = np.empty(self.n_pixels, dtype=np.complex128)
        n = ctypes.c_int64()
        check(self._lib.sf_get_bp(self._h, ptr(img), ctypes.byref(n), SF_MEM_HOST))
        return img, n.value

    def set_pixel_stats(self, B_re, beta, L, pulse_count, fallbacks):
        B = None if B_re is None else _f64(B_re)
        bb = None if beta is None else _c128(beta)
        check(self._lib.sf_set_pixel_stats(self._h, ptr(B), ptr(bb), float(L), int(pulse_count),
                                           int(fallbacks), SF_MEM_HOST))
        self.version += 1

    def set_stats(self, A_re, b, L, pulse_count, fallbacks):
        a = None if A_re is None else _f64(A_re)
        bb = None if b is None else _c128(b)
        if a is not None and a.shape != (self.m_atoms, self.m_atoms):
            raise ValueError("A_re shape mismatch")
        if bb is not None and bb.shape != (self.m_atoms,):
            raise ValueError("b shape mismatch")
        check(self._lib.sf_set_stats(self._h, ptr(a), ptr(bb), float(L), int(pulse_count),
                                     int(fallbacks), SF_MEM_HOST))
        self.version += 1

    def reconstruct(self, c, out=None):
        if hasattr(c, "data_ptr"):
            torch = _torch()
            self._bind()
            if out is None:
                out = torch.empty(self.n_pixels, dtype=torch.float64, device=c.device)
            check(self._lib.sf_reconstruct(self._h, ptr(c), ptr(out), SF_MEM_DEVICE))
            return out
        cc = _f64(c)
        img = np.empty(self.n_pixels, dtype=np.float64)
        check(self._lib.sf_reconstruct(self._h, ptr(cc), ptr(img), SF_MEM_HOST))
        return img

    def profile(self, enable=True):
        """Start (or stop) per-kernel CUDA-event timing on the engine stream."""
        check(self._lib.sf_profile(self._h, 1 if enable else 0))

    def profile_bytes(self):
        """Tile-store bytes the FISTA matvec requested since profile(True)."""
        v = ctypes.c_int64()
        check(self._lib.sf_profile_bytes(self._h, ctypes.byref(v)))
        return v.value

    def profile_read(self, kind):
        """(launches, total_ms) for kind in _lib.K_GEMV/K_GRAM/K_STEP/K_OPERATOR."""
        n = ctypes.c_int64()
        ms = ctypes.c_double()
        check(self._lib.sf_profile_read(self._h, int(kind), ctypes.byref(n), ctypes.byref(ms)))
        return n.value, ms.value

    def timings(self):
        a = ctypes.c_float()
        f = ctypes.c_float()
        check(self._lib.sf_last_timings(self._h, ctypes.byref(a), ctypes.byref(f)))
        return a.value, f.value
