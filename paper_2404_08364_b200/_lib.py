"""ctypes binding of libflowwalk.so (the C ABI in include/flowwalk.h).

There is no CPU fallback: if the shared library is missing or CUDA is not
usable, every walk entry point raises ``FlowWalkUnavailable``.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FW_LIB_PATH") or os.path.join(_HERE, "libflowwalk.so")

FW_OK, FW_EVALIDATION, FW_ECONFIG, FW_ECUDA, FW_ENOMEM, FW_EFORMAT = range(6)
ORDER_AUTO, ORDER_SEQUENTIAL = 0, 1
ST_FIELDS = ("steps", "edges_scanned", "collectives", "draws", "small_tasks",
             "large_tasks", "sampled_steps", "alg_bytes")


class FlowWalkUnavailable(RuntimeError):
    """The CUDA extension is not built or no CUDA device is usable."""


class FwApp(ctypes.Structure):
    _fields_ = [("app_id", ctypes.c_int32), ("weighted", ctypes.c_int32),
                ("length", ctypes.c_uint32), ("schema_len", ctypes.c_uint32),
                ("schema", ctypes.c_void_p), ("stop_prob", ctypes.c_double),
                ("inv_a", ctypes.c_double), ("inv_b", ctypes.c_double)]


class FwEngine(ctypes.Structure):
    _fields_ = [("k_small", ctypes.c_int32), ("k_big", ctypes.c_int32),
                ("d_t", ctypes.c_int64), ("sampler_id", ctypes.c_int32),
                ("order_mode", ctypes.c_int32)]


class FwStats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ST_FIELDS] + [
        ("kernel_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
        ("exact_order", ctypes.c_int32), ("grid_ctas", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32), ("d2h_pieces", ctypes.c_int32),
        ("tail_ms", ctypes.c_double), ("aux_bytes", ctypes.c_int64),
        ("aux_allocations", ctypes.c_int64), ("scratch_bytes", ctypes.c_int64)]


class FwGraphInfo(ctypes.Structure):
    _fields_ = [("max_degree", ctypes.c_int64), ("max_degree_vertex", ctypes.c_int64),
                ("max_weight", ctypes.c_float), ("min_weight_lowbit_exp", ctypes.c_int32),
                ("has_labels", ctypes.c_int32), ("bad_weights", ctypes.c_int32),
                ("sorted_lists", ctypes.c_int32), ("pad_", ctypes.c_int32)]


EXPORTS = ("fw_last_error", "fw_device_count", "fw_graph_create", "fw_graph_create_device",
           "fw_graph_replicate", "fw_graph_destroy", "fw_graph_set_scratch_limit", "fw_graph_info_get", "fw_walk", "fw_walk_device",
           "fw_validate_device", "fw_sampler_trials_device", "fw_rmat_edges_device",
           "fw_synth_weights_device", "fw_synth_labels_device", "fw_edges_max_id",
           "fw_build_csr_device", "fw_fwg1_info", "fw_fwg1_read", "fw_crc32_device")

_lib = None


def load(path=LIB_PATH):
    """Load the library and declare every exported signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FlowWalkUnavailable(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    P, I32, U32, I64, U64, D = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32,
                                ctypes.c_int64, ctypes.c_uint64, ctypes.c_double)
    sig = {
        "fw_last_error": ([], ctypes.c_char_p),
        "fw_device_count": ([P], I32),
        "fw_graph_create": ([P, P, P, P, U64, U64, I32, P], I32),
        "fw_graph_create_device": ([P, P, P, P, U64, U64, I32, P], I32),
        "fw_graph_replicate": ([P, I32, P], I32),
        "fw_graph_destroy": ([P], I32),
        "fw_graph_set_scratch_limit": ([P, U64], I32),
        "fw_graph_info_get": ([P, P], I32),
        "fw_walk": ([P, P, U64, U64, P, P, U64, P, P, P], I32),
        "fw_walk_device": ([P, P, U64, U64, P, P, U64, P, P, P, P], I32),
        "fw_validate_device": ([P, P, U64, P, P, U32, P, U32, P, P], I32),
        "fw_sampler_trials_device": ([I32, P, U32, U32, U64, U64, P, P, D, U32, P, P, P], I32),
        "fw_rmat_edges_device": ([U64, I32, D, D, D, U64, U64, P, P, P], I32),
        "fw_synth_weights_device": ([U64, U64, U64, P, P], I32),
        "fw_synth_labels_device": ([U64, U32, U64, U64, P, P], I32),
        "fw_edges_max_id": ([P, P, U64, P, P], I32),
        "fw_build_csr_device": ([P, P, P, P, U64, U64, P, P, P, P, P], I32),
        "fw_fwg1_info": ([ctypes.c_char_p, P, P, P], I32),
        "fw_fwg1_read": ([ctypes.c_char_p, U64, U64, I32, P, P, P, P, P, P], I32),
        "fw_crc32_device": ([P, U64, P, P], I32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc, msg=None):
    """Map a C status code onto the reference's exception classes.  ``msg``:
    fw_last_error() as read on the thread that made the failing call (the
    message is thread-local)."""
    if rc == FW_OK:
        return
    from .errors import ConfigError, FormatError, ValidationError
    if msg is None:
        msg = load().fw_last_error().decode(errors="replace")
    if rc == FW_EVALIDATION:
        raise ValidationError(msg)
    if rc == FW_ECONFIG:
        raise ConfigError(msg)
    if rc == FW_ENOMEM:
        raise MemoryError(msg)
    if rc == FW_EFORMAT:
        raise FormatError(msg)
    raise RuntimeError(f"flowwalk CUDA error: {msg}")


def device_count():
    lib = load()
    n = ctypes.c_int(0)
    rc = lib.fw_device_count(ctypes.byref(n))
    if rc != FW_OK:
        return 0
    return n.value


def require_device():
    if device_count() < 1:
        raise FlowWalkUnavailable("no CUDA device visible; the walk engine has no CPU path")
