"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the C parity oracle.

``walk`` mirrors the argument values the reference's ``Worker.pass_once``
hands to ``step_pass`` (``engine.py:209-221``): ``inv_a = 1.0 / a`` and
``inv_b = 1.0 / b`` computed in Python float64, the schema only for
MetaPath (``engine.py:165-166``), zero labels for unlabelled graphs
(``graph.py:68-76``), sampler auto-resolution (``engine.py:79-87``).
"""

import ctypes
import os
import subprocess

import numpy as np

MASK64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

APP_IDS = {"deepwalk": 0, "ppr": 1, "node2vec": 2, "metapath": 3}


def mix64(z):
    """rng.py:24-29."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def stream_base(key, sid):
    """rng.py:32-35."""
    h = mix64((key & MASK64) + GOLDEN)
    return mix64(h ^ ((sid & MASK64) * MIX1 & MASK64))


def u01(base, ctr):
    """_kernels.py:63-66 / rng.py:38-41 with the base precomputed."""
    z = mix64((base + (ctr & MASK64) * GOLDEN) & MASK64)
    return (z >> 11) * (1.0 / (1 << 53))


def build():
    """Compile liboracle.so from walk_oracle.c (make, in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def oracle_lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        lib.fwo_walk.argtypes = [P, P, P, P, P, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_uint32,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                 P, ctypes.c_uint32, ctypes.c_int, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                 P, P, P, ctypes.c_int]
        lib.fwo_walk.restype = ctypes.c_int
        lib.fwo_validate.argtypes = [P, P, P, P, ctypes.c_uint64, P, P, ctypes.c_uint32,
                                     P, ctypes.c_uint32]
        lib.fwo_validate.restype = ctypes.c_int64
        lib.fwo_mix64.argtypes = [ctypes.c_uint64]
        lib.fwo_mix64.restype = ctypes.c_uint64
        lib.fwo_stream_base.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.fwo_stream_base.restype = ctypes.c_uint64
        lib.fwo_u01.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.fwo_u01.restype = ctypes.c_double
        _lib = lib
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def resolve_sampler(sampler, app):
    """engine.py:79-87 (SAMPLER_ZPRS = 0, SAMPLER_DPRS = 1)."""
    if sampler == "dprs":
        return 1
    if sampler == "zprs":
        return 0
    return 1 if app == "node2vec" else 0


def walk(offsets, targets, weights, labels, starts, *, app="deepwalk", length=80,
         stop_prob=0.2, a=2.0, b=0.5, schema=(0, 1, 2, 3, 4), weighted=True,
         sampler="auto", k_small=32, k_big=256, degree_threshold=1024, seed=0,
         base_qid=0, threads=None):
    """Replay-mode walks for starts[i] with global qid base_qid + i.

    Returns (sequences (n, length) u32 sentinel-padded, lengths (n,) u32,
    stats int64[6] = steps, edges, collectives, draws, small, large).
    """
    lib = oracle_lib()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.uint32)
    weights = np.ascontiguousarray(weights, dtype=np.float32)
    if labels is not None:
        labels = np.ascontiguousarray(labels, dtype=np.uint8)
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    n = len(starts)
    seq = np.empty((n, length), dtype=np.uint32)
    lens = np.empty(n, dtype=np.uint32)
    stats = np.zeros(6, dtype=np.int64)
    sch = np.ascontiguousarray(schema if app == "metapath" else (), dtype=np.int64)
    if sch.size == 0:
        sch = np.zeros(1, dtype=np.int64)
        sch_len = 0
    else:
        sch_len = len(sch)
    if threads is None:
        threads = os.cpu_count() or 1
    lib.fwo_walk(_ptr(offsets), _ptr(targets), _ptr(weights), _ptr(labels), _ptr(starts),
                 n, base_qid, APP_IDS[app], int(bool(weighted)), length,
                 float(stop_prob), 1.0 / a, 1.0 / b, _ptr(sch), sch_len,
                 resolve_sampler(sampler, app), k_small, k_big, degree_threshold,
                 seed & MASK64, _ptr(seq), _ptr(lens), _ptr(stats), int(threads))
    return seq, lens, stats


def validate(offsets, targets, labels, starts, sequences, lengths, schema=()):
    """validate_walks restatement (_kernels.py:486-546); returns #violations."""
    lib = oracle_lib()
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    targets = np.ascontiguousarray(targets, dtype=np.uint32)
    if labels is not None:
        labels = np.ascontiguousarray(labels, dtype=np.uint8)
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    seq = np.ascontiguousarray(sequences, dtype=np.uint32)
    lens = np.ascontiguousarray(lengths, dtype=np.uint32)
    sch = np.ascontiguousarray(schema, dtype=np.int64)
    sch_len = len(sch)
    if sch_len == 0:
        sch = np.zeros(1, dtype=np.int64)
    return int(lib.fwo_validate(_ptr(offsets), _ptr(targets), _ptr(labels), _ptr(starts),
                                len(starts), _ptr(seq), _ptr(lens), seq.shape[1],
                                _ptr(sch), sch_len))
