"""B200-native engine for the per-pulse Online-FISTA hot path of sparse SAR imaging.

Drop-in for the hot-path API of the reference package ``sarfista``
(arXiv 2603.08582): forward model, edgelet dictionary, and the streaming
``accumulate`` / ``online_fista_pulse`` calls.  All numerical work runs in the
sm_100a kernels of ``libsarfista_b200.so`` behind the C ABI in
``include/sarfista_b200.h``; importing this package does not touch the GPU.
"""

__version__ = "0.1.0"

from . import baseline, dictionary, geometry, harness, metrics, rng, solver
from .engine import Engine

# the reference package's public names, served by the device-backed modules
_PUBLIC = {
    dictionary: ("DictionarySpec EdgeletDictionary EdgeletParams build_dictionary "
                 "build_extended_dictionary compose rasterize_edgelet synthesize"),
    geometry: ("SPEED_OF_LIGHT PulseGeometry SceneGrid TrajectoryConfig angular_frequencies "
               "build_forward_matrix pixel_positions platform_position pulse_at "
               "round_trip_delay trajectory_angle"),
    rng: "counter_uniform counter_unit_complex_vector splitmix64",
    solver: ("GeometricPulse NoiseCovariance PulseMeasurement SolverConfig SolverState "
             "SufficientStatistics accumulate batch_fista hermitian_top_eigenvalue "
             "online_fista_pulse reconstruct soft_threshold"),
    harness: "StreamingRunner TraceRow simulate_echoes simulate_pulse",
    metrics: "Method count_large memory_values snr_db",
}
for _module, _names in _PUBLIC.items():
    for _name in _names.split():
        globals()[_name] = getattr(_module, _name)
__all__ = ["Engine"] + [n for names in _PUBLIC.values() for n in names.split()]
del _module, _names, _name
