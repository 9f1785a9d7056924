"""B200-native engine for the per-pulse Online-FISTA hot path of sparse SAR imaging.

Drop-in for the hot-path API of the reference package ``sarfista``
(arXiv 2603.08582): forward model, edgelet dictionary, and the streaming
``accumulate`` / ``online_fista_pulse`` calls.  All numerical work runs in the
sm_100a kernels of ``libsarfista_b200.so`` behind the C ABI in
``include/sarfista_b200.h``; importing this package does not touch the GPU.
"""

__version__ = "0.1.0"

from .dictionary import (
    DictionarySpec,
    EdgeletDictionary,
    EdgeletParams,
    build_dictionary,
    build_extended_dictionary,
    compose,
    rasterize_edgelet,
    synthesize,
)
from .engine import Engine
from .geometry import (
    SPEED_OF_LIGHT,
    PulseGeometry,
    SceneGrid,
    TrajectoryConfig,
    angular_frequencies,
    build_forward_matrix,
    pixel_positions,
    platform_position,
    pulse_at,
    round_trip_delay,
    trajectory_angle,
)
from .rng import counter_uniform, counter_unit_complex_vector, splitmix64
from .solver import (
    GeometricPulse,
    NoiseCovariance,
    PulseMeasurement,
    SolverConfig,
    SolverState,
    SufficientStatistics,
    accumulate,
    batch_fista,
    hermitian_top_eigenvalue,
    online_fista_pulse,
    reconstruct,
    soft_threshold,
)
from .harness import StreamingRunner, TraceRow, simulate_echoes, simulate_pulse
from .metrics import Method, count_large, memory_values, snr_db
