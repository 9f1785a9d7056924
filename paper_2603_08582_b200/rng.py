"""Counter-based SplitMix64 primitives (reference rng.py:14-37).

The engine derives its power-iteration start vector on the device
(csrc/sf_geom.cu k_start_vector); these host functions expose the same
sequence for API parity (vectorised with wrapping uint64 arithmetic instead of
the reference's per-element Python loop).
"""

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64(state):
    """One SplitMix64 finalisation step (rng.py:14-19); int in, int out."""
    return int(_mix(np.array([int(state) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


def _uniforms(seed, index):
    seed = np.uint64(int(seed) & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        mixed = _mix(seed * _GOLDEN + np.asarray(index, dtype=np.uint64) + np.uint64(1))
    return (mixed >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def counter_uniform(seed, index):
    """Deterministic uniform in [0, 1) for (seed, index) (rng.py:22-25)."""
    return float(_uniforms(seed, np.array([int(index)], dtype=np.uint64))[0])


def counter_unit_complex_vector(n, salt=0x5EED):
    """Unit-norm complex start vector of the power iteration (rng.py:28-37)."""
    n = int(n)
    k = np.arange(n, dtype=np.uint64)
    re = _uniforms(salt, np.uint64(2) * k) - 0.5
    im = _uniforms(salt, np.uint64(2) * k + np.uint64(1)) - 0.5
    v = re + 1j * im
    nrm = np.linalg.norm(v)
    if nrm == 0.0:
        v = np.ones(n, dtype=np.complex128)
        nrm = np.sqrt(float(n))
    return v / nrm
