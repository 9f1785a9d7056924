"""BASELINE.json workloads as seeded synthetic inputs.

Decisions recorded here apply identically to the engine and to the oracle:
  G1  real coefficient vector (the reference loop, solver.py:214-226)
  G2  slant range 10 km at 30 deg elevation -> radius = 1e4 cos 30, altitude
      = 1e4 sin 30; arc [offset, offset + span], every position fires
  G3  identity + every (strided) origin per orientation, clipped atoms kept,
      unit-norm columns (dictionary.build_extended_dictionary)
  G4  lambda_n = lam_rel * max_j |b_n,j| after the pulse's accumulate
  G5  sigma^2 = mean_k,m |F_k rho|^2 / 10^(SNR/10) over the whole run; noise
      CN(0, sigma^2), real then imaginary standard normals (harness.py:229-232)
  G6  cfg3 steps = 10
Truth: complex amplitudes |a| ~ U[0.5, 1.5], arg a ~ U[0, 2 pi) on distinct
identity atoms (points) and distinct edgelet atoms (segments).
Input generation is host-side numpy and is not part of the timed hot path.
"""

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .dictionary import build_extended_dictionary
from .geometry import (
    SceneGrid,
    TrajectoryConfig,
    angular_frequencies,
    pixel_positions,
    platform_position,
)

SPEED_OF_LIGHT = 299_792_458.0


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    side: int
    n_freq: int
    n_pulses: int
    arc_deg: float
    length: int
    n_rot: int
    stride: int
    n_points: int
    n_segments: int
    snr_db: float
    steps: int
    seed: int
    center_hz: float = 10.0e9
    bandwidth_hz: float = 500.0e6
    range_m: float = 10_000.0
    elevation_deg: float = 30.0
    arc_offset_deg: float = 0.0
    lam_rel: float = 0.05

    @property
    def n_pixels(self):
        return self.side * self.side

    @property
    def m_atoms(self):
        per_rot = ((self.side + self.stride - 1) // self.stride) ** 2
        return self.n_pixels + self.n_rot * per_rot


CONFIGS = {
    0: WorkloadConfig("cfg0", 32, 64, 64, 30.0, 4, 4, 1, 6, 2, 20.0, 10, 0),
    1: WorkloadConfig("cfg1", 64, 128, 128, 45.0, 6, 8, 1, 20, 8, 15.0, 10, 1),
    2: WorkloadConfig("cfg2", 32, 64, 64, 30.0, 4, 4, 1, 6, 2, 20.0, 10, 2),
    3: WorkloadConfig("cfg3", 128, 256, 256, 60.0, 8, 4, 1, 60, 24, 15.0, 10, 3),
    4: WorkloadConfig("cfg4", 256, 512, 512, 90.0, 8, 4, 2, 200, 64, 10.0, 5, 4),
}

# Small geometries with the same structure, for parity tests the oracle
# finishes in seconds.
SMALL = {
    "tiny": WorkloadConfig("tiny", 8, 16, 8, 30.0, 3, 4, 1, 3, 1, 20.0, 10, 11),
    "small": WorkloadConfig("small", 16, 32, 24, 30.0, 4, 4, 1, 4, 2, 20.0, 10, 12),
    "small8": WorkloadConfig("small8", 16, 48, 16, 45.0, 5, 8, 1, 5, 2, 15.0, 10, 13),
    "stride2": WorkloadConfig("stride2", 16, 32, 12, 90.0, 4, 4, 2, 4, 2, 10.0, 5, 14),
}


@dataclass
class Workload:
    cfg: WorkloadConfig
    grid: SceneGrid
    dictionary: object
    omega: np.ndarray           # [N_r]
    positions: np.ndarray       # [P][3]
    d: np.ndarray               # [P][N_r] complex
    sigma2: float
    c_true: np.ndarray          # [M] complex
    rho: np.ndarray             # [N] complex
    extra: dict = field(default_factory=dict)

    @property
    def m_atoms(self):
        return self.dictionary.m_atoms


def _ell_apply(idx, w, c, n):
    """rho = H c from the ELL table (host)."""
    out = np.zeros(n, dtype=np.result_type(c.dtype, np.float64))
    mask = idx >= 0
    j = np.nonzero(mask)[0]
    np.add.at(out, idx[mask], w[mask] * c[j])
    return out


def trajectory(cfg):
    el = math.radians(cfg.elevation_deg)
    return TrajectoryConfig(
        radius=cfg.range_m * math.cos(el),
        altitude=cfg.range_m * math.sin(el),
        arc_start=math.radians(cfg.arc_offset_deg),
        arc_end=math.radians(cfg.arc_offset_deg + cfg.arc_deg),
        num_positions=cfg.n_pulses,
    )


def forward_matrix_host(omega, gamma, xyz):
    """Host copy of F for data simulation only (geometry.py:97-107)."""
    diff = xyz - gamma[None, :]
    tau = (2.0 / SPEED_OF_LIGHT) * np.sqrt((diff * diff).sum(axis=1))
    return np.exp(-1j * np.outer(omega, tau))


def generate(cfg, dictionary=None, device_sim=False):
    """Seeded synthetic inputs for one scene.  ``device_sim``: the noise-free
    echoes F_k rho come from the device simulator (sf_simulate_echo, equal to
    the host forward model to ~1e-13 relative); the noise draws are unchanged."""
    grid = SceneGrid(cfg.side, 1.0, (0.0, 0.0, 0.0))
    if dictionary is None:
        dictionary = build_extended_dictionary(cfg.side, cfg.length, cfg.n_rot, cfg.stride)
    n, m = grid.n_pixels, dictionary.m_atoms
    trng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 0]))
    pts = trng.choice(n, size=cfg.n_points, replace=False)
    segs = n + trng.choice(m - n, size=cfg.n_segments, replace=False)
    support = np.concatenate([pts, segs])
    amp = trng.uniform(0.5, 1.5, size=support.size)
    phase = trng.uniform(0.0, 2.0 * math.pi, size=support.size)
    c_true = np.zeros(m, dtype=np.complex128)
    c_true[support] = amp * np.exp(1j * phase)
    rho = _ell_apply(dictionary.ell_idx, dictionary.ell_w, c_true, n)

    omega = angular_frequencies(cfg.n_freq, cfg.center_hz, cfg.bandwidth_hz)
    traj = trajectory(cfg)
    positions = np.stack([platform_position(traj, grid.center, k) for k in range(cfg.n_pulses)])
    xyz = pixel_positions(grid)
    if device_sim:
        from .harness import simulate_echoes

        clean = simulate_echoes(grid, positions, omega, rho)
    else:
        # F_k rho over the pixels rho touches (the others contribute exact zeros)
        nz = np.nonzero(rho)[0]
        clean = np.empty((cfg.n_pulses, cfg.n_freq), dtype=np.complex128)
        for k in range(cfg.n_pulses):
            clean[k] = forward_matrix_host(omega, positions[k], xyz[nz]) @ rho[nz]
    sigma2 = float(np.mean(np.abs(clean) ** 2) / 10.0 ** (cfg.snr_db / 10.0))
    nrng = np.random.default_rng(cfg.seed)
    scale = math.sqrt(sigma2) / math.sqrt(2.0)
    d = np.empty_like(clean)
    for k in range(cfg.n_pulses):
        d[k] = clean[k] + scale * (nrng.standard_normal(cfg.n_freq)
                                   + 1j * nrng.standard_normal(cfg.n_freq))
    return Workload(cfg, grid, dictionary, omega, positions, d, sigma2, c_true, rho)


def generate_batch(cfg, n_scenes, dictionary=None, device_sim=False):
    """cfg2: independent scenes, seed SeedSequence([seed, s]), azimuth offset U[0, 360)."""
    if dictionary is None:
        dictionary = build_extended_dictionary(cfg.side, cfg.length, cfg.n_rot, cfg.stride)
    out = []
    for s in range(n_scenes):
        srng = np.random.default_rng(np.random.SeedSequence([cfg.seed, s]))
        offset = float(srng.uniform(0.0, 360.0))
        seed = int(srng.integers(0, 2**31 - 1))
        out.append(generate(replace(cfg, seed=seed, arc_offset_deg=offset), dictionary, device_sim))
    return out
