"""ctypes binding of ``libsarfista_b200.so`` (the C ABI in include/sarfista_b200.h).

There is no fallback: if the shared library is missing or no sm_100 device is
present, every compute entry point raises.  Status codes map to the exception
types the reference raises for the same conditions (solver.py uses ValueError
for shape/domain errors and RuntimeError for state errors).
"""

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsarfista_b200.so")

SF_OK, SF_EINVAL, SF_ESTATE, SF_ECUDA, SF_ENOMEM, SF_ENCCL, SF_EUNSUPPORTED = range(7)
SF_MEM_HOST, SF_MEM_DEVICE = 0, 1
PRECISIONS = {"tf32x3": 0, "tf32": 1, "fp32": 2, "f16x3": 3, "dirichlet": 4}
K_GEMV, K_GRAM, K_STEP, K_OPERATOR, K_LIPSCHITZ, K_FISTA, K_KTILDE, K_FOLD = range(8)
ABI_VERSION = 3
MODES = {"atom": 0, "pixel": 1}

# every symbol the header declares (checked by tests/test_abi.py)
EXPORTED = (
    "sf_create", "sf_destroy", "sf_set_stream", "sf_synchronize", "sf_reset", "sf_info",
    "sf_accumulate_geom", "sf_accumulate_dense", "sf_fista", "sf_get_scalars",
    "sf_get_power_diag", "sf_probe_store_read", "sf_probe_matvec", "sf_apply_store", "sf_profile_bytes", "sf_pulse_metrics", "sf_get_b",
    "sf_get_A_re", "sf_set_stats", "sf_get_pixel_stats", "sf_set_pixel_stats", "sf_get_bp", "sf_set_bp", "sf_init_device", "sf_get_A", "sf_set_stats_complex", "sf_dense_residual", "sf_tile_store",
    "sf_copy_tiles",
    "sf_reconstruct", "sf_last_timings", "sf_profile",
    "sf_profile_read",
    "sf_plan_shard", "sf_nccl_unique_id", "sf_shard_init", "sf_loopback_create",
    "sf_loopback_destroy", "sf_shard_init_loopback", "sf_shard_sizes", "sf_peer_create",
    "sf_peer_blob_size", "sf_peer_export", "sf_peer_import", "sf_peer_destroy",
    "sf_shard_init_peer",
    "sf_delay_phase_matrix", "sf_fista_inner", "sf_hermitian_top_eigenvalue",
    "sf_compose_ell", "sf_soft_threshold", "sf_simulate_echo", "sf_last_error", "sf_abi_version",
    "sf_launch_count", "sf_accumulate_geom_batch", "sf_get_batch_scalars", "sf_batch_lipschitz",
)


class SfDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("m_atoms", ctypes.c_int64),
        ("n_freq", ctypes.c_int32),
        ("ell_width", ctypes.c_int32),
        ("n_pixels", ctypes.c_int64),
        ("ell_idx", ctypes.c_void_p),
        ("ell_w", ctypes.c_void_p),
        ("pixel_xyz", ctypes.c_void_p),
        ("precision", ctypes.c_int32),
        ("power_max_iter", ctypes.c_int32),
        ("l_floor", ctypes.c_double),
        ("power_rel_tol", ctypes.c_double),
        ("mode", ctypes.c_int32),
        ("batch", ctypes.c_int32),
        ("keep_complex", ctypes.c_int32),
    ]


_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_D = ctypes.c_double

_SIGNATURES = {
    "sf_create": [ctypes.POINTER(SfDesc), ctypes.POINTER(_P)],
    "sf_destroy": [_P],
    "sf_set_stream": [_P, _P],
    "sf_synchronize": [_P],
    "sf_reset": [_P, _D],
    "sf_info": [_P, _P, _P, _P, _P],
    "sf_accumulate_geom": [_P, _P, _P, _P, _D, _I32],
    "sf_accumulate_dense": [_P, _P, _P, _I32, _D, _I32],
    "sf_fista": [_P, _P, _P, _I32, _D, _D, _I32, _D, _P],
    "sf_get_scalars": [_P, _P, _P, _P, _P],
    "sf_get_power_diag": [_P, _P],
    "sf_probe_store_read": [_P, _I32, _P],
    "sf_probe_matvec": [_P, _I32, _I32, _P],
    "sf_apply_store": [_P, _P, _P, _I32],
    "sf_profile_bytes": [_P, _P],
    "sf_pulse_metrics": [_P, _P, _P, _P, ctypes.c_double, _P],
    "sf_get_b": [_P, _P, _I32],
    "sf_get_A_re": [_P, _P, _I32],
    "sf_set_stats": [_P, _P, _P, _D, _I64, _I64, _I32],
    "sf_get_pixel_stats": [_P, _P, _P, _I32],
    "sf_set_pixel_stats": [_P, _P, _P, _D, _I64, _I64, _I32],
    "sf_get_bp": [_P, _P, _P, _I32],
    "sf_set_bp": [_P, _P, _I32],
    "sf_init_device": [_I32],
    "sf_get_A": [_P, _P, _I32],
    "sf_set_stats_complex": [_P, _P, _P, ctypes.c_double, _I64, _I64, _I32],
    "sf_dense_residual": [_I32, _P, _P, _I32, _I64, _P, ctypes.c_double, _P, _P],
    "sf_tile_store": [_P, _P, _P, _P],
    "sf_copy_tiles": [_P, _P, _I32, _I32],
    "sf_reconstruct": [_P, _P, _P, _I32],
    "sf_last_timings": [_P, _P, _P],
    "sf_profile": [_P, _I32],
    "sf_profile_read": [_P, _I32, _P, _P],
    "sf_plan_shard": [_I64, _I32, _I32, _P, _P, _P],
    "sf_nccl_unique_id": [_P],
    "sf_shard_init": [_P, _I32, _I32, _P],
    "sf_loopback_create": [_I32, _P],
    "sf_loopback_destroy": [_P],
    "sf_shard_init_loopback": [_P, _I32, _P],
    "sf_shard_sizes": [_P, _P, _P],
    "sf_peer_create": [_I32, _I32, _I32, _I64, _I64, _P, _P],
    "sf_peer_export": [_P, _P],
    "sf_peer_import": [_P, _P],
    "sf_peer_destroy": [_P],
    "sf_shard_init_peer": [_P, _P],
    "sf_delay_phase_matrix": [_I32, _P, _I32, _P, _I64, _P],
    "sf_fista_inner": [_I32, _P, _P, _P, _I64, _D, _D, _D, _I32, _P, _P],
    "sf_hermitian_top_eigenvalue": [_I32, _P, _I64, _D, _I32, _P, _P],
    "sf_compose_ell": [_I32, _P, _I32, _I64, _P, _P, _I64, _I32, _P],
    "sf_soft_threshold": [_I32, _P, _I64, _I32, _D, _P],
    "sf_simulate_echo": [_I32, _P, _I32, _P, _I32, _P, _P, _I64, _P],
    "sf_accumulate_geom_batch": [_P, _P, _P, _P, _P, _I32],
    "sf_get_batch_scalars": [_P, _P, _P, _P],
    "sf_batch_lipschitz": [_P, _P, _P, _P, _I32, _D, _I32, _P, _P],
}


def load():
    """Load the engine library once; raise if it is absent (no fallback path)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` or "
                "`python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        lib.sf_last_error.argtypes = []
        lib.sf_last_error.restype = ctypes.c_char_p
        lib.sf_abi_version.argtypes = []
        lib.sf_abi_version.restype = ctypes.c_int32
        lib.sf_launch_count.argtypes = []
        lib.sf_launch_count.restype = ctypes.c_int64
        lib.sf_peer_blob_size.argtypes = []
        lib.sf_peer_blob_size.restype = ctypes.c_int64
        lib.sf_peer_destroy.restype = None
        if lib.sf_abi_version() != ABI_VERSION:
            raise ImportError("libsarfista_b200.so ABI version mismatch; rebuild it")
        _lib = lib
        return lib


def check(status):
    """Raise the Python exception matching an sf_status."""
    if status == SF_OK:
        return
    msg = load().sf_last_error().decode("utf-8", "replace")
    if status == SF_EINVAL:
        raise ValueError(msg)
    if status == SF_ESTATE:
        raise RuntimeError(msg)
    if status == SF_ENOMEM:
        raise MemoryError(msg)
    if status == SF_EUNSUPPORTED:
        raise RuntimeError("unsupported device: " + msg)
    raise RuntimeError(f"sarfista_b200 error {status}: {msg}")


def ptr(a):
    """Raw address of a numpy array or torch tensor (no copies are made here)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


def launch_count():
    return int(load().sf_launch_count())
