"""Drop-in ``sarfista``: the reference package with its per-pulse hot path on
the B200 engine.

Put ``dropin/`` first on ``sys.path`` (``PYTHONPATH=dropin``) and
``import sarfista`` resolves here.  The modules on the hot path
are this repository's, registered under the reference's module names:

  sarfista.solver      paper_2603_08582_b200.solver  (accumulate, online_fista_pulse,
                       statistics types, power iteration, soft threshold, batch
                       oracle, checkpoints)
  sarfista.kernels     the plugin seam (kernels.py:27-116) on the device
  sarfista.geometry    paper_2603_08582_b200.geometry (forward model)
  sarfista.dictionary  paper_2603_08582_b200.dictionary (edgelets, compose)
  sarfista.rng         paper_2603_08582_b200.rng

Everything else -- scene construction, the experiment harness, metrics,
sampling schedules, the BP baseline, image IO and the CLI (out of
scope) -- is the reference's own source, loaded from the installed reference
package (``baseline/_ref/sarfista``, or ``$SARFISTA_REFERENCE_DIR``) as
submodules of this package, so its relative imports (``from .solver import
accumulate``) bind to the engine.  Without the reference install only the
hot-path modules are available.
"""

import importlib.util
import os
import sys
import types

_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(os.path.dirname(_HERE))
if _REPO not in sys.path:
    sys.path.insert(0, _REPO)

from paper_2603_08582_b200 import dictionary as _dictionary  # noqa: E402
from paper_2603_08582_b200 import geometry as _geometry  # noqa: E402
from paper_2603_08582_b200 import kernels as _kdev  # noqa: E402
from paper_2603_08582_b200 import rng as _rng  # noqa: E402
from paper_2603_08582_b200 import solver as _solver  # noqa: E402

__version__ = "0.1.0"

REFERENCE_DIR = os.environ.get("SARFISTA_REFERENCE_DIR",
                               os.path.join(_REPO, "baseline", "_ref", "sarfista"))


def _seam_module():
    """kernels.py's public names.  There is one implementation of each kernel
    (the device one); the reference's per-backend names resolve to it and its
    optional numba backend reports as not built."""
    k = types.ModuleType(__name__ + ".kernels", _kdev.__doc__)
    k.delay_phase_matrix = k.delay_phase_matrix_numpy = _kdev.delay_phase_matrix
    k.fista_inner = k.fista_inner_numpy = _kdev.fista_inner
    k.delay_phase_matrix_numba = None
    k.fista_inner_numba = None
    k.NUMBA_REQUESTED = os.environ.get("SARFISTA_NUMBA", "1").strip() != "0"
    k.NUMBA_ACTIVE = False
    return k


kernels = _seam_module()
solver = _solver
geometry = _geometry
dictionary = _dictionary
rng = _rng
for _name, _mod in (("kernels", kernels), ("solver", solver), ("geometry", geometry),
                    ("dictionary", dictionary), ("rng", rng)):
    sys.modules[f"{__name__}.{_name}"] = _mod


def _load_reference(name):
    path = os.path.join(REFERENCE_DIR, name + ".py")
    spec = importlib.util.spec_from_file_location(f"{__name__}.{name}", path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    globals()[name] = mod
    return mod


HAVE_REFERENCE = os.path.isfile(os.path.join(REFERENCE_DIR, "harness.py"))
if HAVE_REFERENCE:
    # dependency order of the reference's relative imports
    for _name in ("scene", "baseline", "metrics", "sampling", "imgio", "harness", "cli"):
        _load_reference(_name)

def _init_device():
    """Create the device context at import (as importing numpy/numba does its
    set-up), so a caller's first timed call does not pay it; silent without a GPU."""
    try:
        from paper_2603_08582_b200 import _lib

        _lib.load().sf_init_device(0)
    except Exception:
        pass


_init_device()

from paper_2603_08582_b200.dictionary import (  # noqa: E402
    DictionarySpec,
    EdgeletDictionary,
    EdgeletParams,
    build_dictionary,
    compose,
    rasterize_edgelet,
    synthesize,
)
from paper_2603_08582_b200.geometry import (  # noqa: E402
    SPEED_OF_LIGHT,
    PulseGeometry,
    TrajectoryConfig,
    angular_frequencies,
    build_forward_matrix,
    platform_position,
    pulse_at,
    round_trip_delay,
)
from paper_2603_08582_b200.solver import (  # noqa: E402
    NoiseCovariance,
    PulseMeasurement,
    SolverConfig,
    SolverState,
    SufficientStatistics,
    accumulate,
    batch_fista,
    batch_gradient,
    batch_objective,
    hermitian_top_eigenvalue,
    load_checkpoint,
    online_fista_pulse,
    reconstruct,
    save_checkpoint,
    soft_threshold,
)

if HAVE_REFERENCE:
    from .baseline import BpAccumulator, bp_accumulate, bp_image_db, bp_image_linear  # noqa: E402,F401
    from .harness import (  # noqa: E402,F401
        ExperimentConfig,
        ExperimentTrace,
        StreamingRunner,
        load_config,
        run_experiment,
        simulate_pulse,
    )
    from .metrics import Method, MemoryReport, SnrReport, count_large, memory_values, snr_db  # noqa: E402,F401,E501
    from .sampling import PulseSchedule, bernoulli_schedule, required_pulses, rip_constant  # noqa: E402,F401,E501
    from .scene import (  # noqa: E402,F401
        IDEAL_COEFF_COUNTS,
        SceneGrid,
        SceneId,
        ideal_components,
        make_scene,
        pixel_position,
        pixel_positions,
    )
else:
    from paper_2603_08582_b200.geometry import SceneGrid, pixel_positions  # noqa: E402,F401
