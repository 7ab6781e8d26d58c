"""The walk API: drop-in for reswalk.engine (run_batches / run, engine.py:263-364).

What stays the same as the reference
  * signatures, dataclasses (EngineConfig, BatchResult, RunStats), validation
    order and exception classes (engine.py:64-77, 271-283), Eq. 3 batch
    sizing (engine.py:90-105), sentinel-padded (count, L) uint32 sequences
    (start vertex not stored), FWR1 result files (engine.py:382-421);
  * replay-mode results, bit for bit: every query is a pure function of
    (graph, seed, global qid, app, k_small, k_big, d_t, sampler).

What changes
  * the CPU worker threads / local pools / numba step_pass are replaced by
    one persistent sm_100a kernel per device (libflowwalk.so, csrc/), whose
    warps pull queries from an atomic cursor;
  * the graph is uploaded once through pinned staging, checked on the device
    (offsets, target range, per-vertex sortedness), and cached across calls
    on the same host ``Graph`` object (``evict`` drops it; ``to_device`` /
    ``DeviceGraph`` give an explicitly resident graph);
  * ``EngineConfig.devices`` replicates the graph on several GPUs and splits
    each batch's query range across them (no collective on the walk path);
  * ``replay=False`` (the reference's schedule-dependent free-run keying)
    maps to replay keying: the GPU is always deterministic;
  * ``workers``/``local_pool``/``meter``/``on_pass`` are CPU-scheduler hooks
    with no device counterpart; they are accepted and ignored (``on_pass``
    warns once).  RunStats.small_tasks/large_tasks carry the routing info.
There is no CPU fallback: without the CUDA library every call raises.
"""

import struct
import threading
import time
import warnings
import weakref
import zlib
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .apps import APP_IDS, AppConfig
from .errors import ConfigError, FormatError, ValidationError

RESULT_SENTINEL = np.uint32(0xFFFFFFFF)
SAMPLER_ZPRS, SAMPLER_DPRS = 0, 1
RESULT_MAGIC = b"FWR1"


class AllocationMeter:
    """API twin of engine.py:35-48 (host-side scratch accounting)."""

    def __init__(self):
        self.total_bytes = 0
        self.allocations = 0
        self.by_tag = {}

    def register(self, tag, arr):
        self.total_bytes += arr.nbytes
        self.allocations += 1
        self.by_tag[tag] = self.by_tag.get(tag, 0) + arr.nbytes
        return arr


@dataclass
class EngineConfig:
    workers: int = 1
    k_small: int = 32
    k_big: int = 256
    local_pool: int = 64
    degree_threshold: int = 1024
    memory_budget: int | None = None
    graph_bytes: int | None = None
    vertex_bytes: int = 4
    replay: bool = False
    sampler: str = "auto"
    devices: tuple = (0,)        # B200 extension: GPUs holding a graph replica
    order: str = "auto"          # fp64 summation order: auto | sequential

    def validate(self):
        if self.workers < 1:
            raise ConfigError("need at least one worker")
        if self.local_pool < 1:
            raise ConfigError("local pool must hold at least one query")
        if self.degree_threshold < 1:
            raise ConfigError("degree threshold must be >= 1")
        if not 1 <= self.k_small <= self.k_big:
            raise ConfigError("lane widths must satisfy 1 <= k_small <= k_big")
        if self.k_big > 1000:
            raise ConfigError("k_big larger than the stream-id lane field")
        if self.sampler not in ("auto", "zprs", "dprs"):
            raise ConfigError(f"unknown sampler {self.sampler!r}")
        if self.order not in ("auto", "sequential"):
            raise ConfigError(f"unknown order {self.order!r}")
        if len(self.devices) < 1:
            raise ConfigError("need at least one device")
        return self

    def resolve_sampler(self, app):
        """engine.py:79-87: node2vec defaults to the single-scan DPRS."""
        if self.sampler == "dprs":
            return SAMPLER_DPRS
        if self.sampler == "zprs":
            return SAMPLER_ZPRS
        return SAMPLER_DPRS if app == "node2vec" else SAMPLER_ZPRS


def batch_size(cfg, l_max):
    """Eq. 3 (engine.py:90-105)."""
    if cfg.memory_budget is None:
        raise ConfigError("no memory budget configured")
    m_graph = cfg.graph_bytes or 0
    if cfg.memory_budget <= m_graph:
        raise ConfigError(
            f"memory budget {cfg.memory_budget} does not exceed graph size {m_graph}")
    size = (cfg.memory_budget - m_graph) // (2 * (l_max + 1) * cfg.vertex_bytes)
    if size < 1:
        raise ConfigError("memory budget too small for a single query")
    return int(size)


class GlobalPool:
    """Host twin of engine.py:108-128 (the device uses an atomic cursor)."""

    def __init__(self, starts, base_qid=0):
        self.starts = starts
        self.base_qid = base_qid
        self.cursor = 0
        self._lock = threading.Lock()

    def fetch(self, want):
        if want < 1:
            raise ValidationError("fetch wants at least one query")
        with self._lock:
            lo = self.cursor
            hi = min(lo + want, len(self.starts))
            self.cursor = hi
        return [(self.base_qid + i, int(self.starts[i])) for i in range(lo, hi)]

    def remaining(self):
        return len(self.starts) - self.cursor


@dataclass
class BatchResult:
    batch_index: int
    base_qid: int
    count: int
    sequences: np.ndarray  # (count, l_max) uint32, sentinel padded
    lengths: np.ndarray    # (count,) uint32


@dataclass
class RunStats:
    queries: int = 0
    batches: int = 0
    steps: int = 0
    edges_scanned: int = 0
    collectives: int = 0
    draws: int = 0
    small_tasks: int = 0
    large_tasks: int = 0
    elapsed_s: float = 0.0
    aux_bytes: int = 0
    aux_allocations: int = 0
    completed: int = 0
    per_worker_completed: list = field(default_factory=list)
    completed_query_ids: np.ndarray | None = None
    # device extensions
    sampled_steps: int = 0
    alg_bytes: int = 0
    kernel_ms: float = 0.0
    exact_order: bool = False  # tree-order scans ran (modes "exact" and "certified")
    # "sequential": the reference's summation order replayed; "exact": every
    # partial sum exact, tree scans; "certified": tree scans with certified
    # accept tests, ambiguous steps re-run in order
    summation: str = "sequential"


# ---------------------------------------------------------------------------
# Device graph handles
# ---------------------------------------------------------------------------
class _Handle:
    def __init__(self, ptr, device, keepalive=None):
        self.ptr = ptr
        self.device = device
        self._keep = keepalive

    def close(self):
        if self.ptr:
            _lib.load().fw_graph_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self):
        out = _lib.FwGraphInfo()
        _lib.check(_lib.load().fw_graph_info_get(self.ptr, _ctypes_ref(out)))
        return out


def _ctypes_ref(obj):
    import ctypes
    return ctypes.byref(obj)


def _upload(g, device):
    """fw_graph_create: host checks (Graph.validate, graph.py:70-81), then one
    pinned-staged H2D of the CSR arrays and the device-side CSR check."""
    import ctypes
    lib = _lib.load()
    if hasattr(g, "validate"):
        g.validate()
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    tgt = np.ascontiguousarray(g.targets, dtype=np.uint32)
    w = np.ascontiguousarray(g.weights, dtype=np.float32)
    lab = None if getattr(g, "labels", None) is None else np.ascontiguousarray(g.labels, np.uint8)
    if g.max_degree() >= 1 << 32:
        raise ConfigError("vertex degree >= 2^32 is not supported")
    out = ctypes.c_void_p()
    _lib.check(lib.fw_graph_create(off.ctypes.data, tgt.ctypes.data, w.ctypes.data,
                                   None if lab is None else lab.ctypes.data,
                                   g.vertex_count, g.edge_count, device, ctypes.byref(out)))
    return _Handle(out.value, device)


def _replica_handle(src, device):
    """fw_graph_replicate: device-to-device peer copies of a resident CSR."""
    import ctypes
    out = ctypes.c_void_p()
    _lib.check(_lib.load().fw_graph_replicate(src.ptr, device, ctypes.byref(out)))
    return _Handle(out.value, device)


# Device replicas of host Graphs, kept across run() calls (the reference
# re-reads its numpy arrays every call; re-uploading 18 GB per call at s27
# would dominate).  Keyed by the Graph object (weakly: a dropped graph frees
# its replicas); a fingerprint of the array addresses, sizes and a strided
# sample of the contents detects a graph whose arrays were replaced or edited
# in place.  ``evict(g)`` releases a graph's replicas explicitly.
_CACHE = weakref.WeakKeyDictionary()
_CACHE_LOCK = threading.Lock()


def _fingerprint(g):
    fp = [int(g.vertex_count), int(g.edge_count)]
    for a in (g.offsets, g.targets, g.weights, getattr(g, "labels", None)):
        if a is None:
            fp.append(None)
            continue
        a = np.asarray(a)
        step = max(1, a.size // 4096)
        sample = np.ascontiguousarray(a.reshape(-1)[::step][:4096])
        fp.append((a.__array_interface__["data"][0], a.nbytes, str(a.dtype),
                   zlib.crc32(memoryview(sample).cast("B"))))
    return tuple(fp)


def _cached_handles(g, devices):
    fp = _fingerprint(g)
    with _CACHE_LOCK:
        entry = _CACHE.get(g)
        if entry is None or entry[0] != fp:
            if entry is not None:
                for h in entry[1].values():
                    h.close()
            entry = (fp, {})
            _CACHE[g] = entry
        reps = entry[1]
        for d in devices:
            if d in reps:
                continue
            reps[d] = _replica_handle(next(iter(reps.values())), d) if reps else _upload(g, d)
        return [reps[d] for d in devices]


def evict(g):
    """Release the device replicas cached for host graph ``g``."""
    with _CACHE_LOCK:
        entry = _CACHE.pop(g, None)
    if entry is not None:
        for h in entry[1].values():
            h.close()


class DeviceGraph:
    """A CSR resident in HBM (torch tensors as the allocator), reusable
    across calls.  Arrays: offsets int64, targets int32 (bit-cast uint32),
    weights float32, labels uint8 or None.  targets/weights must stay
    readable 16 bytes past their end (the walk kernel loads 16-byte tiles);
    to_device() and rmat_graph_device() allocate that padding."""

    def __init__(self, vertex_count, edge_count, offsets, targets, weights, labels=None,
                 device=0):
        import ctypes
        self.vertex_count = int(vertex_count)
        self.edge_count = int(edge_count)
        self.offsets, self.targets, self.weights, self.labels = offsets, targets, weights, labels
        self.device = device
        out = ctypes.c_void_p()
        lib = _lib.load()
        _lib.check(lib.fw_graph_create_device(
            offsets.data_ptr(), targets.data_ptr(), weights.data_ptr(),
            None if labels is None else labels.data_ptr(), self.vertex_count,
            self.edge_count, device, ctypes.byref(out)))
        self._handle = _Handle(out.value, device, keepalive=(offsets, targets, weights, labels))
        self._replicas = {device: self._handle}
        self._info = self._handle.info()

    def handle(self, device):
        if device not in self._replicas:
            self._replicas[device] = _replicate(self, device)
        return self._replicas[device]

    def max_degree(self):
        return int(self._info.max_degree)

    def max_degree_vertex(self):
        return int(self._info.max_degree_vertex)

    def degree(self, v):
        return int((self.offsets[v + 1] - self.offsets[v]).item())

    @property
    def nbytes(self):
        n = 8 * (self.vertex_count + 1) + 8 * self.edge_count
        return n + (self.edge_count if self.labels is not None else 0)

    def to_host(self):
        from .graph import Graph
        return Graph(self.vertex_count, self.edge_count, self.offsets.cpu().numpy(),
                     self.targets.cpu().numpy().view(np.uint32), self.weights.cpu().numpy(),
                     None if self.labels is None else self.labels.cpu().numpy())

    def close(self):
        for h in self._replicas.values():
            h.close()
        self._replicas.clear()


def _replicate(dg, device):
    """A replica of a resident CSR on `device` (fw_graph_replicate: NVLink
    peer copies when the devices are peers)."""
    return _replica_handle(dg._handle, device)


def to_device(g, device=0):
    """Upload a host Graph once and keep it resident (DeviceGraph)."""
    import torch
    dev = torch.device("cuda", device)
    def tg(a, dt, pad=0):
        host = torch.from_numpy(np.ascontiguousarray(a).view(dt))
        out = torch.empty(host.numel() + pad, dtype=host.dtype, device=dev)[:host.numel()]
        out.copy_(host)
        return out

    lab = None if g.labels is None else tg(np.asarray(g.labels, np.uint8), np.uint8)
    return DeviceGraph(g.vertex_count, g.edge_count, tg(np.asarray(g.offsets, np.int64), np.int64),
                       tg(np.asarray(g.targets, np.uint32), np.int32, 4),
                       tg(np.asarray(g.weights, np.float32), np.float32, 4), lab, device=device)


class _Session:
    """Per-call device state: one graph handle per configured device.  Host
    graphs go through the replica cache; a DeviceGraph's handles are the
    caller's (borrowed).  Nothing is released at close."""

    def __init__(self, g, eng_cfg):
        _lib.load()
        _lib.require_device()
        self.devices = tuple(eng_cfg.devices)
        if isinstance(g, DeviceGraph):
            self.handles = [g.handle(d) for d in self.devices]
        else:
            self.handles = _cached_handles(g, self.devices)

    def close(self):
        pass


def _fw_structs(app_cfg, eng_cfg):
    app_id = APP_IDS[app_cfg.app]
    schema = np.ascontiguousarray(app_cfg.schema if app_cfg.app == "metapath" else (),
                                  dtype=np.int64)
    app = _lib.FwApp(app_id=app_id, weighted=int(bool(app_cfg.weighted)),
                     length=app_cfg.length, schema_len=len(schema),
                     schema=schema.ctypes.data if len(schema) else None,
                     stop_prob=float(app_cfg.stop_prob),
                     inv_a=1.0 / app_cfg.a, inv_b=1.0 / app_cfg.b)
    eng = _lib.FwEngine(k_small=eng_cfg.k_small, k_big=eng_cfg.k_big,
                        d_t=eng_cfg.degree_threshold,
                        sampler_id=eng_cfg.resolve_sampler(app_cfg.app),
                        order_mode=_lib.ORDER_SEQUENTIAL if eng_cfg.order == "sequential"
                        else _lib.ORDER_AUTO)
    return app, eng, schema


def _walk_batch(sess, starts, base_qid, app, eng, seed, seq, lens, totals):
    """Split one batch's query range over the session's devices (one host
    thread per device; ctypes releases the GIL)."""
    n = len(starts)
    parts = len(sess.handles)
    bounds = [n * i // parts for i in range(parts + 1)]
    lib = _lib.load()
    results = [None] * parts

    def one(i):
        lo, hi = bounds[i], bounds[i + 1]
        st = _lib.FwStats()
        rc = lib.fw_walk(sess.handles[i].ptr, starts[lo:].ctypes.data if hi > lo else None,
                         hi - lo, base_qid + lo, _ctypes_ref(app), _ctypes_ref(eng),
                         seed & 0xFFFFFFFFFFFFFFFF,
                         seq[lo * app.length:].ctypes.data if hi > lo else None,
                         lens[lo:].ctypes.data if hi > lo else None, _ctypes_ref(st))
        # fw_last_error is thread-local: read it on the calling thread
        msg = lib.fw_last_error().decode(errors="replace") if rc else ""
        results[i] = (rc, msg, st, hi - lo)

    if parts == 1:
        one(0)
    else:
        with ThreadPoolExecutor(max_workers=parts) as ex:
            list(ex.map(one, range(parts)))
    batch_ms = 0.0
    aux = 0
    for i, (rc, msg, st, cnt) in enumerate(results):
        _lib.check(rc, msg)
        for f in _lib.ST_FIELDS:
            totals[f] += getattr(st, f)
        batch_ms = max(batch_ms, st.kernel_ms)  # devices run concurrently
        aux += st.aux_bytes
        totals["aux_allocations"] = max(totals["aux_allocations"], st.aux_allocations)
        totals["per_device"][i] += cnt
        totals["exact_order"] = bool(st.exact_order)
        totals["summation"] = _SUMMATION.get(int(st.exact_order), "sequential")
    totals["kernel_ms"] += batch_ms  # batches run one after another
    totals["aux_bytes"] = max(totals["aux_bytes"], aux)


_SUMMATION = {0: "sequential", 1: "exact", 2: "certified"}


def _new_totals(parts=1):
    t = {f: 0 for f in _lib.ST_FIELDS}
    t["kernel_ms"] = 0.0
    t["exact_order"] = False
    t["summation"] = "sequential"
    t["aux_bytes"] = 0
    t["aux_allocations"] = 0
    t["per_device"] = [0] * parts
    return t


def run_batches(g, starts, app_cfg, eng_cfg, seed=0, workers=None, meter=None,
                on_pass=None, *, base_qid=0, _totals=None):
    """Generator over BatchResult, double-buffered (engine.py:263-322).

    Batch b+1 is walked on the device(s) by a driver thread while the
    consumer holds batch b; each BatchResult's arrays are views into one of
    two reused buffers, valid until the generator is resumed twice.

    ``base_qid`` (B200 extension, keyword-only): global id of starts[0].  In
    replay mode a walk is a pure function of its global qid, so a caller
    that shards one query set (one process per GPU) passes its shard's
    offset and gets exactly its slice of the unsharded run.
    """
    app_cfg.validate()
    eng_cfg.validate()
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    if len(starts) and (starts.min() < 0 or starts.max() >= g.vertex_count):
        raise ValidationError("start vertex out of range")
    if app_cfg.length >= 1 << 20:
        raise ConfigError("walk length exceeds the replay stream-id field")
    if on_pass is not None:
        warnings.warn("on_pass is a CPU-scheduler hook; the device engine never calls it",
                      RuntimeWarning, stacklevel=2)
    n = len(starts)
    size = batch_size(eng_cfg, app_cfg.length) if eng_cfg.memory_budget is not None else max(n, 1)
    n_batches = (n + size - 1) // size if n else 0
    if base_qid < 0 or base_qid + n >= 1 << 33:
        raise ConfigError("query ids exceed the replay stream-id field")
    l_max = app_cfg.length
    totals = _totals if _totals is not None else _new_totals(len(eng_cfg.devices))
    if n_batches == 0:
        return
    app, eng, _schema = _fw_structs(app_cfg, eng_cfg)
    sess = _Session(g, eng_cfg)
    rows = min(size, n)
    # the second buffer only exists when there is a second batch
    buffers = [(np.empty(rows * l_max, np.uint32), np.empty(rows, np.uint32))
               for _ in range(min(2, n_batches))]

    def compute(b, buf):
        seq, lens = buf
        base = b * size
        count = min(size, n - base)
        _walk_batch(sess, starts[base:base + count], base_qid + base, app, eng, seed, seq, lens,
                    totals)
        return BatchResult(batch_index=b, base_qid=base_qid + base, count=count,
                           sequences=seq[:count * l_max].reshape(count, l_max),
                           lengths=lens[:count])

    driver = ThreadPoolExecutor(max_workers=1)
    try:
        pending = driver.submit(compute, 0, buffers[0])
        for b in range(n_batches):
            res = pending.result()
            if b + 1 < n_batches:
                pending = driver.submit(compute, b + 1, buffers[(b + 1) % 2])
            yield res
    finally:
        driver.shutdown(wait=True)
        sess.close()


def run(g, starts, app_cfg, eng_cfg, seed=0, sink=None, keep_query_ids=False, on_pass=None,
        *, base_qid=0):
    """Execute all queries; returns RunStats (engine.py:325-364)."""
    app_cfg.validate()
    eng_cfg.validate()
    totals = _new_totals(len(eng_cfg.devices))
    t0 = time.perf_counter()
    batches = 0
    for batch in run_batches(g, starts, app_cfg, eng_cfg, seed, on_pass=on_pass,
                             base_qid=base_qid, _totals=totals):
        batches += 1
        if sink is not None:
            sink(batch)
    elapsed = time.perf_counter() - t0
    n = len(starts)
    stats = RunStats(
        queries=n, batches=batches, steps=int(totals["steps"]),
        edges_scanned=int(totals["edges_scanned"]), collectives=int(totals["collectives"]),
        draws=int(totals["draws"]), small_tasks=int(totals["small_tasks"]),
        large_tasks=int(totals["large_tasks"]), elapsed_s=elapsed,
        # the library's own device scratch (cursor slots, counters, piece
        # counters, schema copies), summed over devices: independent of d_max
        # and |Q|, like the reference's metered aux bytes
        aux_bytes=int(totals["aux_bytes"]), aux_allocations=int(totals["aux_allocations"]),
        completed=n, per_worker_completed=_per_worker(totals["per_device"], eng_cfg.workers),
        sampled_steps=int(totals["sampled_steps"]), alg_bytes=int(totals["alg_bytes"]),
        kernel_ms=float(totals["kernel_ms"]), exact_order=bool(totals["exact_order"]),
        summation=totals["summation"])
    if keep_query_ids:
        stats.completed_query_ids = np.arange(base_qid, base_qid + n, dtype=np.int64)
    return stats


def _per_worker(per_device, workers):
    """RunStats.per_worker_completed has one entry per configured worker
    (engine.py:357).  The device engine has no CPU workers: device d's
    completed queries are spread evenly over the workers w with
    w % len(devices) == d (sum and length match the reference's)."""
    out = [0] * workers
    nd = len(per_device)
    for d, cnt in enumerate(per_device):
        ws = [w for w in range(workers) if w % nd == d] or [d % workers]
        for j, w in enumerate(ws):
            out[w] += cnt * (j + 1) // len(ws) - cnt * j // len(ws)
    return out


def throughput_report(stats):
    elapsed = max(stats.elapsed_s, 1e-9)
    return {
        "elapsed_s": stats.elapsed_s,
        "edges_per_sec": stats.edges_scanned / elapsed,
        "steps_per_sec": stats.steps / elapsed,
        "edges_scanned": stats.edges_scanned,
        "steps": stats.steps,
        "collectives": stats.collectives,
        "batches": stats.batches,
    }


def write_result_file(path, g, starts, app_cfg, eng_cfg, seed=0):
    """FWR1: magic, <QI (count, l_max), then per query u32 length + row."""
    l_max = app_cfg.length
    with open(path, "wb") as fh:
        fh.write(RESULT_MAGIC)
        fh.write(struct.pack("<QI", len(starts), l_max))

        def sink(batch):
            rows = np.empty((batch.count, 1 + l_max), np.uint32)
            rows[:, 0] = batch.lengths
            rows[:, 1:] = batch.sequences
            fh.write(rows.tobytes())

        return run(g, starts, app_cfg, eng_cfg, seed=seed, sink=sink)


def read_result_file(path):
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 16 or blob[:4] != RESULT_MAGIC:
        raise FormatError(f"{path}: bad magic (not a walk result file)")
    count, l_max = struct.unpack_from("<QI", blob, 4)
    if len(blob) != 16 + count * (1 + l_max) * 4:
        raise FormatError(f"{path}: truncated result file")
    rows = np.frombuffer(blob, dtype="<u4", offset=16).reshape(count, 1 + l_max)
    return rows[:, 0].copy(), rows[:, 1:].copy()
