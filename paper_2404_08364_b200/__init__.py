"""B200-native FlowWalker walk engine: a drop-in for the reference ``reswalk``
walk API (reswalk/__init__.py:15-31) whose hot path -- the dynamic-weight
walk step with DPRS/ZPRS parallel reservoir sampling -- runs as hand-written
sm_100a CUDA (csrc/) behind the C ABI in include/flowwalk.h.

Exports follow reswalk's names for the walk path.  The sampler object layer
(LaneGroup, dprs, zprs, its, alias, rjs), statistics and CLI of the
reference are out of scope.
"""

from .apps import APP_IDS, APPS, AppConfig, WalkQuery
from .engine import (AllocationMeter, BatchResult, DeviceGraph, EngineConfig, GlobalPool,
                     RunStats, batch_size, evict, read_result_file, run, run_batches,
                     throughput_report, to_device, write_result_file)
from .errors import (CapacityError, ConfigError, FormatError, ParseError,
                     RejectionExhausted, ReswalkError, ValidationError)
from .graph import (EdgeList, Graph, build_csr, build_csr_device, load_binary,
                    load_binary_device, parse_edge_list,
                    random_edge_list, save_binary, star_edge_list, synthesize_labels,
                    synthesize_weights)
from .rng import RngStream, make_stream

__version__ = "0.1.0"

__all__ = [
    "APPS", "APP_IDS", "AppConfig", "WalkQuery", "AllocationMeter", "BatchResult",
    "DeviceGraph", "EngineConfig", "GlobalPool", "RunStats", "batch_size", "evict",
    "read_result_file", "run", "run_batches", "throughput_report", "to_device",
    "write_result_file", "CapacityError", "ConfigError", "FormatError", "ParseError",
    "RejectionExhausted", "ReswalkError", "ValidationError", "EdgeList", "Graph",
    "build_csr", "build_csr_device", "load_binary", "load_binary_device", "parse_edge_list", "random_edge_list", "save_binary",
    "star_edge_list", "synthesize_labels", "synthesize_weights", "RngStream", "make_stream",
    "__version__",
]
