"""Drop-in API behaviour on the GPU: FWR1 result files, result batching when
results exceed the device budget, the device-graph cache, CSR validation in
the C ABI, replicas, concurrent launches, base_qid sharding and RunStats
bookkeeping.  Every walk is compared against the golden vectors (generated
by running the reference) or the C oracle."""

import ctypes

import numpy as np
import pytest

import oracle
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import _lib, engine, rmat

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")


def _graph(golden, gname):
    off, tgt, w, lab = golden.graph(gname)
    return fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)


def _run(g, starts, app_cfg, eng_cfg, seed=0, **kw):
    seqs, lens = [], []

    def sink(b):
        seqs.append(b.sequences.copy())
        lens.append(b.lengths.copy())

    st = fw.run(g, starts, app_cfg, eng_cfg, seed=seed, sink=sink, **kw)
    return np.concatenate(seqs), np.concatenate(lens), st


@pytest.fixture(scope="module")
def s16():
    return rmat.rmat_graph(16)


def _golden_case(golden, name):
    case = golden.cases[name]
    app = dict(case["app"])
    if "schema" in app:
        app["schema"] = tuple(app["schema"])
    return case, fw.AppConfig(**app), fw.EngineConfig(replay=True, **case["eng"])


@pytest.mark.parametrize("budget", [None, 2 * 25 * 4 * 300])
def test_fwr1_result_file_roundtrip_equals_golden(golden, tmp_path, budget):
    """write_result_file -> read_result_file (FWR1, engine.py:382-421) gives
    the reference's golden paths, in one batch or in Eq. 3 batches."""
    case, app, eng = _golden_case(golden, "n2v_rmat12")
    if budget is not None:
        eng.memory_budget, eng.graph_bytes = budget, 0
    g = _graph(golden, case["graph"])
    p = tmp_path / "walks.fwr"
    st = fw.write_result_file(p, g, golden.starts("n2v_rmat12"), app, eng, seed=case["seed"])
    lengths, seqs = fw.read_result_file(p)
    want_seq, want_len, want_stats = golden.expected("n2v_rmat12")
    np.testing.assert_array_equal(lengths, want_len)
    np.testing.assert_array_equal(seqs, want_seq)
    assert [getattr(st, f) for f in STAT_NAMES] == want_stats.tolist()
    assert st.batches == (1 if budget is None else -(-len(want_len) // 300))
    blob = bytearray(p.read_bytes())
    with pytest.raises(fw.FormatError):
        (tmp_path / "bad.fwr").write_bytes(b"XXXX" + bytes(blob[4:]))
        fw.read_result_file(tmp_path / "bad.fwr")
    with pytest.raises(fw.FormatError):
        (tmp_path / "short.fwr").write_bytes(bytes(blob[:-4]))
        fw.read_result_file(tmp_path / "short.fwr")


@pytest.mark.parametrize("app", [dict(app="node2vec", length=40, a=2.0, b=0.5),
                                 dict(app="ppr", length=40, stop_prob=0.2)])
def test_device_scratch_limit_sub_launches_bit_exact(s16, app):
    """Results larger than the device scratch budget are walked in
    sub-launches over two alternating device buffers (D2H of one overlapping
    the next launch); the host arrays equal one unbatched oracle run."""
    g = s16
    starts = np.arange(g.vertex_count, dtype=np.int64)
    app_cfg = fw.AppConfig(**app)
    a, e, _schema = engine._fw_structs(app_cfg, fw.EngineConfig(replay=True))
    h = engine._replica_handle(engine._cached_handles(g, (0,))[0], 0)  # a private handle
    lib = _lib.load()
    try:
        per_q = app_cfg.length * 4 + 4 + 8
        _lib.check(lib.fw_graph_set_scratch_limit(h.ptr, per_q * 9000))  # 7 sub-launches
        seq = np.full(len(starts) * app_cfg.length, 7, np.uint32)
        ln = np.full(len(starts), 7, np.uint32)
        st = _lib.FwStats()
        _lib.check(lib.fw_walk(h.ptr, starts.ctypes.data, len(starts), 0, ctypes.byref(a),
                               ctypes.byref(e), 11, seq.ctypes.data, ln.ctypes.data,
                               ctypes.byref(st)))
    finally:
        h.close()
    assert st.kernel_launches == -(-len(starts) // 4500)
    assert st.scratch_bytes <= per_q * 9000
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, seed=11,
                                 **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq.reshape(len(starts), -1), oseq)
    assert [st.steps, st.edges_scanned, st.collectives, st.draws, st.small_tasks,
            st.large_tasks] == ost.tolist()


def test_graph_cache_reuses_and_detects_changes(golden):
    case, app, eng = _golden_case(golden, "n2v_rmat12")
    g = _graph(golden, case["graph"])
    starts = golden.starts("n2v_rmat12")
    want_seq, want_len, _ = golden.expected("n2v_rmat12")
    s1, l1, _ = _run(g, starts, app, eng, case["seed"])
    h1 = engine._cached_handles(g, (0,))[0]
    s2, l2, _ = _run(g, starts, app, eng, case["seed"])
    assert engine._cached_handles(g, (0,))[0] is h1  # no second upload
    np.testing.assert_array_equal(s1, want_seq)
    np.testing.assert_array_equal(s2, want_seq)
    # edit the weights in place: the fingerprint changes, the graph is re-uploaded
    g.weights[:] = np.float32(1.0)
    s3, l3, _ = _run(g, starts, app, eng, case["seed"])
    assert engine._cached_handles(g, (0,))[0] is not h1
    oseq, oln, _ = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts,
                               app="node2vec", length=app.length, a=app.a, b=app.b,
                               seed=case["seed"], k_small=eng.k_small, k_big=eng.k_big,
                               degree_threshold=eng.degree_threshold)
    np.testing.assert_array_equal(s3, oseq)
    np.testing.assert_array_equal(l3, oln)
    fw.evict(g)
    assert g not in engine._CACHE


def _tiny(off, tgt):
    off = np.asarray(off, np.int64)
    tgt = np.asarray(tgt, np.uint32)
    return off, tgt, np.ones(len(tgt), np.float32)


@pytest.mark.parametrize("bad", ["target", "offsets", "ends"])
def test_c_abi_rejects_malformed_csr(bad):
    """fw_graph_create / fw_graph_create_device check the CSR on the device
    (Graph.validate, graph.py:70-81) instead of faulting in the walk."""
    import torch
    off, tgt, w = _tiny([0, 2, 3, 4], [1, 2, 0, 0])
    if bad == "target":
        tgt[1] = 3
    elif bad == "offsets":
        off[1], off[2] = 3, 2
    else:
        off[3] = 5
    lib = _lib.load()
    out = ctypes.c_void_p()
    rc = lib.fw_graph_create(off.ctypes.data, tgt.ctypes.data, w.ctypes.data, None, 3,
                             len(tgt), 0, ctypes.byref(out))
    assert rc == _lib.FW_EVALIDATION
    d = [torch.from_numpy(x.view(np.int32) if x.dtype == np.uint32 else x).cuda()
         for x in (off, tgt, w)]
    rc = lib.fw_graph_create_device(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), None,
                                    3, len(tgt), 0, ctypes.byref(out))
    assert rc == _lib.FW_EVALIDATION
    g = fw.Graph(3, len(tgt), off, tgt, w)
    with pytest.raises(fw.ValidationError):
        fw.run(g, np.array([0]), fw.AppConfig(app="deepwalk", length=3),
               fw.EngineConfig(replay=True))


def test_unsorted_lists_rejected_for_node2vec_only():
    off, tgt, w = _tiny([0, 3, 4, 5, 6], [3, 1, 2, 0, 0, 0])  # N(0) unsorted
    g = fw.Graph(4, len(tgt), off, tgt, w)
    info = engine._cached_handles(g, (0,))[0].info()
    assert info.sorted_lists == 0
    starts = np.zeros(50, np.int64)
    seq, ln, st = _run(g, starts, fw.AppConfig(app="deepwalk", length=6),
                       fw.EngineConfig(replay=True), 2)
    oseq, oln, _ = oracle.walk(off, tgt, w, None, starts, app="deepwalk", length=6, seed=2)
    np.testing.assert_array_equal(seq, oseq)
    with pytest.raises(fw.ValidationError):
        fw.run(g, starts, fw.AppConfig(app="node2vec", length=6), fw.EngineConfig(replay=True))
    fw.evict(g)


def test_replica_handle_walks_identically(golden):
    """fw_graph_replicate (device-to-device copy; same device here, NVLink
    peers on a multi-GPU node) gives a handle whose walks equal the source's."""
    case, app, eng = _golden_case(golden, "n2v_rmat12")
    dg = fw.to_device(_graph(golden, case["graph"]))
    rep = engine._replicate(dg, 0)
    assert rep.ptr != dg.handle(0).ptr
    assert rep.info().max_degree == dg.max_degree() and rep.info().sorted_lists == 1
    dg._replicas[0] = rep  # walk through the replica
    seq, ln, st = _run(dg, golden.starts("n2v_rmat12"), app, eng, case["seed"])
    want_seq, want_len, want_stats = golden.expected("n2v_rmat12")
    np.testing.assert_array_equal(seq, want_seq)
    np.testing.assert_array_equal(ln, want_len)
    dg.close()


def test_many_concurrent_device_launches_on_two_streams(s16):
    """fw_walk_device launches on two streams, more than the 64 cursor slots:
    a slot is reused only after its previous kernel finished, so no launch
    shares a cursor with a running one (each query walked exactly once)."""
    import torch
    g = s16
    dg = fw.to_device(g)
    h = dg.handle(0).ptr
    lib = _lib.load()
    app_cfg = fw.AppConfig(app="node2vec", length=12)
    a, e, _schema = engine._fw_structs(app_cfg, fw.EngineConfig(replay=True))
    n, L, launches = 512, 12, 150
    starts = torch.arange(n, dtype=torch.int64, device="cuda") * 7 % g.vertex_count
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    seqs = [torch.empty(n * L, dtype=torch.int32, device="cuda") for _ in range(launches)]
    lens = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(launches)]
    stats = torch.zeros(launches, 10, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    for i in range(launches):
        _lib.check(lib.fw_walk_device(h, starts.data_ptr(), n, 1000 * i, ctypes.byref(a),
                                      ctypes.byref(e), 3, seqs[i].data_ptr(), lens[i].data_ptr(),
                                      stats[i].data_ptr(), streams[i % 2].cuda_stream))
    torch.cuda.synchronize()
    st = starts.cpu().numpy()
    for i in (0, 63, 64, 65, 128, 149):
        oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, None, st, app="node2vec",
                                     length=L, seed=3, base_qid=1000 * i)
        np.testing.assert_array_equal(lens[i].cpu().numpy().view(np.uint32), oln)
        np.testing.assert_array_equal(seqs[i].cpu().numpy().view(np.uint32).reshape(n, L), oseq)
        assert stats[i, :6].cpu().numpy().tolist() == ost.tolist()
    dg.close()


def test_base_qid_shard_equals_slice_of_full_run(s16):
    starts = np.arange(6000, dtype=np.int64) * 5 % s16.vertex_count
    app = fw.AppConfig(app="node2vec", length=30)
    full, fl, _ = _run(s16, starts, app, fw.EngineConfig(replay=True), 4)
    part, pl, st = _run(s16, starts[2500:4100], app, fw.EngineConfig(replay=True), 4,
                        base_qid=2500)
    np.testing.assert_array_equal(part, full[2500:4100])
    np.testing.assert_array_equal(pl, fl[2500:4100])


def test_runstats_bookkeeping(s16):
    """aux_bytes is the library's metered scratch (independent of |Q|);
    per_worker_completed has one entry per configured worker (engine.py:357);
    kernel_ms over several batches is their sum."""
    app = fw.AppConfig(app="metapath", length=5, schema=(0, 1, 2, 3, 4))
    eng = fw.EngineConfig(replay=True, workers=3)
    _, _, st1 = _run(s16, np.arange(100, dtype=np.int64), app, eng)
    _, _, st2 = _run(s16, np.arange(60000, dtype=np.int64), app, eng)
    assert 0 < st1.aux_bytes == st2.aux_bytes < 1 << 20
    assert st1.aux_allocations >= 2
    assert len(st2.per_worker_completed) == 3 and sum(st2.per_worker_completed) == 60000
    budget = fw.EngineConfig(replay=True, memory_budget=2 * 6 * 4 * 20000, graph_bytes=0)
    _, _, st3 = _run(s16, np.arange(60000, dtype=np.int64), app, budget)
    assert st3.batches == 3 and st3.kernel_ms > 0


@pytest.mark.parametrize("schema_len", [5, 16, 23])
def test_metapath_schema_inline_and_device_copy(s16, schema_len):
    """Schemas of up to 16 labels ride in the kernel arguments, longer ones
    in a per-slot device copy; both give the oracle's walks."""
    rs = np.random.default_rng(schema_len)
    schema = tuple(int(x) for x in rs.integers(0, 5, schema_len))
    app = dict(app="metapath", length=schema_len, schema=schema)
    starts = rs.integers(0, s16.vertex_count, 20000).astype(np.int64)
    seq, ln, st = _run(s16, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True), 6)
    oseq, oln, ost = oracle.walk(s16.offsets, s16.targets, s16.weights, s16.labels, starts,
                                 seed=6, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
