"""The streaming caller of the hot path (reference harness.py:221-334).

``StreamingRunner.process`` is the reference's per-pulse driver
(harness.py:282-304): accumulate -> online_fista_pulse -> back-projection ->
image -> metrics.  Here accumulate/FISTA run in the engine, the back-projection
accumulator is a by-product of pixel-space accumulate (no dense forward matrix
on the host), and the image is synthesized on the device.

``simulate_pulse`` mirrors harness.py:221-234: d = F rho plus circular complex
Gaussian noise.  F rho is evaluated on the device (sf_simulate_echo); the noise
keeps the reference's host numpy draws (real, then imaginary standard normals)
so the data stream is the reference's to rounding.
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, ptr
from .baseline import BpAccumulator, bp_accumulator, bp_image_linear
from .geometry import PulseGeometry, pixel_positions
from .metrics import Method, PulseMetrics, count_large, memory_values, snr_db
from .solver import (
    GeometricPulse,
    NoiseCovariance,
    SolverConfig,
    SolverState,
    accumulate,
    online_fista_pulse,
    reconstruct,
)


def simulate_echoes(grid, positions, frequencies, rho=None, device=0):
    """Noise-free echoes d_k = F_k rho for platform positions [P][3] -> [P][N_r] (device)."""
    pos = np.ascontiguousarray(np.atleast_2d(positions), dtype=np.float64)
    if pos.ndim != 2 or pos.shape[1] != 3:
        raise ValueError("positions must be (P, 3)")
    omega = np.ascontiguousarray(frequencies, dtype=np.float64)
    r = grid.reflectivity if rho is None else rho
    r = np.ascontiguousarray(np.asarray(r, dtype=np.complex128))
    if r.shape != (grid.n_pixels,):
        raise ValueError("reflectivity length must equal the pixel count")
    xyz = np.ascontiguousarray(pixel_positions(grid))
    out = np.empty((pos.shape[0], omega.shape[0]), dtype=np.complex128)
    check(_lib.load().sf_simulate_echo(int(device), ptr(omega), omega.shape[0], ptr(pos),
                                       pos.shape[0], ptr(xyz), ptr(r), grid.n_pixels, ptr(out)))
    return out


def simulate_pulse(grid, pulse, dictionary, sigma, rng):
    """One pulse of data (harness.py:221-234) as a GeometricPulse.

    Returns (measurement, None): the dense forward matrix the reference returns
    for its back-projection is not materialized -- the engine folds F^H d into
    its device BP accumulator during accumulate().
    """
    d = simulate_echoes(grid, pulse.position, pulse.frequencies)[0]
    if sigma > 0.0:
        scale = sigma / math.sqrt(2.0)
        d = d + scale * (rng.standard_normal(d.size) + 1j * rng.standard_normal(d.size))
    return GeometricPulse(d, pulse, NoiseCovariance.from_sigma(sigma), grid, dictionary), None


@dataclass
class TraceRow:
    pulse_index: int
    n_large: int
    snr_online_db: float
    snr_bp_db: float
    gain_db: float
    memory_online: int
    memory_batch: int


class StreamingRunner:
    """Solver + baseline state of one run; pulses go in one at a time (harness.py:254-334).

    ``cfg`` is anything with ``solver_config()``, ``l_floor``,
    ``large_coeff_threshold`` (the reference's ExperimentConfig; ``converged``
    also reads ``ideal_coeff_count``, ``strict_count_termination`` and
    ``residual_tol``), or a SolverConfig (then ``large_coeff_threshold``
    defaults to 2e-2).

    Geometric pulses (pixel-space engine): each row's metrics are reduced on the
    device from the engine's c, image H c, BP sum and the resident truth
    (metrics.PulseMetrics, sf_pulse_metrics) -- no per-pulse c_hat round trip.
    Dense pulses keep the reference's host evaluation (their BP needs the
    caller's forward matrix).
    """

    def __init__(self, cfg, grid, dictionary, truth=None, **engine_kw):
        self.cfg = cfg
        self.grid = grid
        self.dictionary = dictionary
        if isinstance(cfg, SolverConfig):
            self.solver_cfg = cfg
            self.threshold = 2e-2
        else:
            self.solver_cfg = cfg.solver_config()
            self.threshold = getattr(cfg, "large_coeff_threshold", 2e-2)
        self.state = SolverState.initial(dictionary.m_atoms, self.solver_cfg.l_floor,
                                         dictionary=dictionary, grid=grid, **engine_kw)
        self.truth = np.asarray(grid.reflectivity if truth is None else truth)
        self.truth_mask = np.abs(self.truth) > 0.0
        self.truth_norm = float(np.linalg.norm(self.truth))
        self._bp_host = BpAccumulator.empty(grid.n_pixels)
        self._metrics = None  # device truth / mask, created with the first pixel-mode pulse
        self._last = None     # the last pulse's device sums

    def _device_sums(self):
        stats = self.state.stats
        eng = stats.engine
        if eng is None or eng.mode != "pixel":
            return None
        if self._metrics is None:
            self._metrics = PulseMetrics(self.truth, stats.device, mask=self.truth_mask)
        return self._metrics.evaluate(eng, self.state.c_device(stats.device), self.threshold)

    def process(self, forward, measurement, pulse_index):
        """Accumulate, update the estimate, update BP, and emit one metric row
        (harness.py:282-304; hot lines 284-287)."""
        stats = accumulate(self.state.stats, measurement)
        self.state = online_fista_pulse(
            SolverState(self.state.c_device(self.state.stats.device), self.state.momentum_t,
                        stats), self.solver_cfg)
        m, n = self.dictionary.m_atoms, self.grid.n_pixels
        nr = measurement.d.shape[0]
        sums = self._device_sums()
        self._last = sums
        if sums is not None:
            n_large = sums.n_large
            snr_online = sums.snr_online().snr_db
            snr_bp = sums.snr_bp().snr_db
        else:  # dense pulses: host BP from the caller's forward matrix (baseline.py:23-33)
            if forward is None:
                raise ValueError("dense pulses need the forward matrix for back-projection")
            self._bp_host = BpAccumulator(self._bp_host.image_sum + np.conj(np.asarray(forward)).T
                                          @ np.asarray(measurement.d), self._bp_host.pulse_count + 1)
            recon = reconstruct(self.state, self.dictionary)
            n_large = count_large(self.state.c_hat, self.threshold)
            snr_online = snr_db(recon, self.truth_mask).snr_db
            snr_bp = snr_db(bp_image_linear(self._bp_host), self.truth_mask).snr_db
        return TraceRow(
            pulse_index=pulse_index,
            n_large=n_large,
            snr_online_db=snr_online,
            snr_bp_db=snr_bp,
            gain_db=snr_online - snr_bp,
            memory_online=memory_values(Method.ONLINE_FISTA, m, n, nr, pulse_index).values_stored,
            memory_batch=memory_values(Method.BATCH_FISTA, m, n, nr, pulse_index).values_stored,
        )

    def residual(self):
        """||H c - truth|| / ||truth|| (harness.py:306-310), reduced on the device
        for pixel-space engines."""
        sums = self._device_sums()
        if sums is not None:
            r = math.sqrt(sums.residual_sq)
            return r if self.truth_norm == 0.0 else r / self.truth_norm
        recon = reconstruct(self.state, self.dictionary)
        if self.truth_norm == 0.0:
            return float(np.linalg.norm(recon))
        return float(np.linalg.norm(recon - self.truth)) / self.truth_norm

    def converged(self):
        """The ideal active-atom count, optionally guarded by the residual
        (harness.py:312-318)."""
        sums = self._device_sums()
        n_large = sums.n_large if sums is not None else count_large(self.state.c_hat,
                                                                     self.threshold)
        if n_large != self.cfg.ideal_coeff_count:
            return False
        if getattr(self.cfg, "strict_count_termination", False):
            return True
        return self.residual() <= self.cfg.residual_tol

    def reconstruction(self):
        return reconstruct(self.state, self.dictionary)

    @property
    def bp(self):
        """The back-projection accumulator (harness.py:288): read from the
        device for pixel-space engines, host-side for dense pulses."""
        eng = self.state.stats.engine
        if eng is not None and eng.mode == "pixel":
            return bp_accumulator(self.state.stats)
        return self._bp_host

    def bp_linear(self):
        acc = self.bp
        if acc.pulse_count < 1:
            return np.zeros(self.grid.n_pixels)
        return bp_image_linear(acc)
