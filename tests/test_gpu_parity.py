"""Parity of the sm_100a walk kernel (through the public API and the C ABI)
against the reference's golden vectors and the CPU oracle."""

import numpy as np
import pytest

import oracle
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import rmat

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")


def _graph(golden, gname):
    off, tgt, w, lab = golden.graph(gname)
    return fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)


def _run(g, starts, app_cfg, eng_cfg, seed):
    seqs, lens = [], []

    def sink(b):
        seqs.append(b.sequences.copy())
        lens.append(b.lengths.copy())

    st = fw.run(g, starts, app_cfg, eng_cfg, seed=seed, sink=sink)
    return np.concatenate(seqs), np.concatenate(lens), st


def _cases():
    from conftest import Golden
    return sorted(Golden().cases)


@pytest.mark.parametrize("order", ["auto", "sequential"])
@pytest.mark.parametrize("name", _cases())
def test_golden_bit_exact(golden, name, order):
    case = golden.cases[name]
    g = _graph(golden, case["graph"])
    app = dict(case["app"])
    if "schema" in app:
        app["schema"] = tuple(app["schema"])
    eng = fw.EngineConfig(replay=True, order=order, **case["eng"])
    seq, ln, st = _run(g, golden.starts(name), fw.AppConfig(**app), eng, case["seed"])
    want_seq, want_len, want_stats = golden.expected(name)
    np.testing.assert_array_equal(ln, want_len)
    np.testing.assert_array_equal(seq, want_seq)
    assert [getattr(st, f) for f in STAT_NAMES] == want_stats.tolist()
    assert st.sampled_steps == int(want_len.sum())


@pytest.fixture(scope="module")
def s16():
    return rmat.rmat_graph(16)


@pytest.mark.parametrize("app", [
    dict(app="deepwalk", length=80),
    dict(app="node2vec", length=80, a=2.0, b=0.5),
    dict(app="ppr", length=80, stop_prob=0.2),
    dict(app="metapath", length=5, schema=(0, 1, 2, 3, 4)),
])
def test_rmat_s16_matches_oracle(s16, app):
    """BASELINE config 1 shape (R-MAT s16 ef16, every vertex a query)."""
    g = s16
    starts = np.arange(g.vertex_count, dtype=np.int64)
    if app["app"] == "ppr":
        starts = np.full(20000, g.max_degree_vertex(), np.int64)
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True), 0)
    kw = dict(app)
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, **kw)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
    assert st.exact_order
    sch = app.get("schema", ()) if app["app"] == "metapath" else ()
    assert oracle.validate(g.offsets, g.targets, g.labels, starts, seq, ln, sch) == 0


@pytest.mark.parametrize("scale", [1, 9, 14])
def test_device_rmat_equals_host(scale):
    import torch
    h = rmat.rmat_graph(scale)
    d = rmat.rmat_graph_device(scale)
    np.testing.assert_array_equal(d.offsets.cpu().numpy(), h.offsets)
    np.testing.assert_array_equal(d.targets.cpu().numpy().view(np.uint32), h.targets)
    np.testing.assert_array_equal(d.weights.cpu().numpy(), h.weights)
    np.testing.assert_array_equal(d.labels.cpu().numpy(), h.labels)
    assert d.max_degree() == h.max_degree()
    assert d.max_degree_vertex() == h.max_degree_vertex()
    del torch


def test_device_graph_walk_and_validator():
    import ctypes

    import torch

    from paper_2404_08364_b200 import _lib
    d = rmat.rmat_graph_device(15)
    h = d.to_host()
    n = d.vertex_count
    starts = torch.arange(n, dtype=torch.int64, device="cuda")
    L = 40
    seq = torch.empty(n * L, dtype=torch.int32, device="cuda")
    ln = torch.empty(n, dtype=torch.int32, device="cuda")
    stats = torch.zeros(10, dtype=torch.int64, device="cuda")
    app = fw.AppConfig(app="node2vec", length=L)
    eng = fw.EngineConfig()
    from paper_2404_08364_b200.engine import _fw_structs
    a, e, _s = _fw_structs(app, eng)
    lib = _lib.load()
    stream = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.fw_walk_device(d.handle(0).ptr, starts.data_ptr(), n, 0, ctypes.byref(a),
                                  ctypes.byref(e), 0, seq.data_ptr(), ln.data_ptr(),
                                  stats.data_ptr(), stream))
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.check(lib.fw_validate_device(d.handle(0).ptr, starts.data_ptr(), n, seq.data_ptr(),
                                      ln.data_ptr(), L, None, 0, bad.data_ptr(), stream))
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    oseq, oln, ost = oracle.walk(h.offsets, h.targets, h.weights, h.labels,
                                 np.arange(n), app="node2vec", length=L)
    np.testing.assert_array_equal(ln.cpu().numpy().view(np.uint32), oln)
    np.testing.assert_array_equal(seq.cpu().numpy().view(np.uint32).reshape(n, L), oseq)
    st = stats.cpu().numpy()
    assert st[:6].tolist() == ost.tolist()
    assert st[6] == int(oln.sum())
    # corrupt one step: the GPU validator must see it
    s2 = seq.view(n, L).clone()
    i = int(np.flatnonzero(oln >= 3)[0])
    s2[i, 2] = int(s2[i, 2].item() == 0)
    bad.zero_()
    _lib.check(lib.fw_validate_device(d.handle(0).ptr, starts.data_ptr(), n, s2.data_ptr(),
                                      ln.data_ptr(), L, None, 0, bad.data_ptr(), stream))
    torch.cuda.synchronize()
    assert int(bad.item()) >= 0  # may be a real edge by chance; checked exactly below
    want = oracle.validate(h.offsets, h.targets, h.labels, np.arange(n),
                           s2.cpu().numpy().view(np.uint32), oln)
    assert int(bad.item()) == want


def test_split_across_device_handles(golden):
    """EngineConfig.devices: the query range is split across graph replicas;
    global qids keep the result identical (here two replicas on one GPU)."""
    g = _graph(golden, "rmat12")
    starts = golden.starts("n2v_rmat12")
    eng = fw.EngineConfig(replay=True, devices=(0, 0, 0))
    seq, ln, st = _run(g, starts, fw.AppConfig(app="node2vec", length=24), eng, 0)
    want_seq, want_len, want_stats = golden.expected("n2v_rmat12")
    np.testing.assert_array_equal(seq, want_seq)
    np.testing.assert_array_equal(ln, want_len)
    assert [getattr(st, f) for f in STAT_NAMES] == want_stats.tolist()


def test_base_qid_window_equals_slice(s16):
    """A query recomputed from its global qid equals its slot in a full run
    (replay makes a walk a pure function of the global qid)."""
    g = s16
    starts = np.arange(4096, dtype=np.int64)
    app = fw.AppConfig(app="node2vec", length=30)
    full, fl, _ = _run(g, starts, app, fw.EngineConfig(replay=True), 3)
    budget = fw.EngineConfig(replay=True, memory_budget=2 * 31 * 4 * 1000, graph_bytes=0)
    part, pl, st = _run(g, starts, app, budget, 3)
    assert st.batches == 5
    np.testing.assert_array_equal(part, full)
    np.testing.assert_array_equal(pl, fl)


def test_errors_raise_before_kernel(s16):
    with pytest.raises(fw.ValidationError):
        list(fw.run_batches(s16, np.array([s16.vertex_count]), fw.AppConfig(),
                            fw.EngineConfig()))
    with pytest.raises(fw.ConfigError):
        list(fw.run_batches(s16, np.array([0]), fw.AppConfig(length=1 << 20),
                            fw.EngineConfig()))
    with pytest.raises(fw.ConfigError):
        fw.EngineConfig(k_big=1001).validate()


@pytest.mark.parametrize("gather", ["direct", "nccl"])
def test_torchrun_two_ranks_strong_scaling_gather(tmp_path, gather):
    """bench.py's multi-rank path end to end: 2 ranks (sharing this box's GPU,
    gloo for the control collectives), CSR generated on rank 0 and
    broadcast, qids partitioned (strong scaling), path segments gathered to
    rank 0 -- either written straight into rank 0's buffer by every rank's
    walk kernel (CUDA IPC, "direct") or sent point to point after the walk
    ("nccl" mode; gloo here) -- the gathered paths must equal one oracle run
    over all qids."""
    import json
    import os
    import subprocess
    import sys

    from paper_2404_08364_b200 import rmat
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    out = tmp_path / "gather.npz"
    n = 6000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(root, "bench.py"), "--gpus", "2", "--scale", "14", "--nq", str(n),
           "--steps", "1", "--warmup", "1",
           "--dump-gather", str(out), "--no-cpu-baseline", "--no-e2e", "--length", "24",
           "--gather", gather]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stderr[-3000:]
    line = json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["queries_per_gpu"] == n // 2
    assert line["run"]["gather"] == gather and line["run"]["gather_ms"] is not None
    assert len(line["run"]["per_rank_walk_ms"]) == 2
    z = np.load(out)
    g = rmat.rmat_graph(14, labels=False)
    starts = np.arange(n, dtype=np.int64) % g.vertex_count
    oseq, oln, _ = oracle.walk(g.offsets, g.targets, g.weights, None, starts,
                               app="node2vec", length=24)
    np.testing.assert_array_equal(z["lens"], oln)
    np.testing.assert_array_equal(z["seq"], oseq)


def _trial_cases():
    from conftest import Golden
    return [c["name"] for c in Golden().trials]


@pytest.mark.parametrize("name", _trial_cases())
def test_sampler_trials_bit_exact(golden, name):
    """GPU trial kernels == the reference's numba trial kernels
    (_kernels.py:84-277): picks, collectives per task, rejection rounds."""
    from paper_2404_08364_b200 import trials
    case = next(c for c in golden.trials if c["name"] == name)
    w = golden.z[f"t_w_{case['vec']}"]
    res = trials.run_trials(case["sampler"], w, case["trials"], int(case["seed"]), k=case["k"])
    np.testing.assert_array_equal(res.picks, golden.z[f"t_picks_{name}"])
    key = f"t_aux_{name}"
    if key in golden.z:
        aux = res.collectives if res.collectives is not None else res.rounds
        np.testing.assert_array_equal(aux, golden.z[key])


def test_device_graph_reusable_across_calls(golden):
    """A resident DeviceGraph survives run() calls (handles are borrowed)."""
    g = _graph(golden, "rmat12")
    dg = fw.to_device(g)
    starts = golden.starts("n2v_rmat12")
    app = fw.AppConfig(app="node2vec", length=24)
    for _ in range(2):
        seq, ln, _st = _run(dg, starts, app, fw.EngineConfig(replay=True), 0)
        want_seq, want_len, _ = golden.expected("n2v_rmat12")
        np.testing.assert_array_equal(seq, want_seq)
        np.testing.assert_array_equal(ln, want_len)


def _chi2_pass(counts, probs, alpha=1e-3):
    """Pearson chi-square with bins of expected count < 5 pooled."""
    from scipy.stats import chi2
    n = counts.sum()
    exp = probs * n
    order = np.argsort(exp)
    obs_p, exp_p, acc_o, acc_e = [], [], 0.0, 0.0
    for i in order:
        acc_o += counts[i]
        acc_e += exp[i]
        if acc_e >= 5:
            obs_p.append(acc_o)
            exp_p.append(acc_e)
            acc_o = acc_e = 0.0
    if acc_e > 0 and exp_p:
        obs_p[-1] += acc_o
        exp_p[-1] += acc_e
    obs_p, exp_p = np.array(obs_p), np.array(exp_p)
    stat = float(((obs_p - exp_p) ** 2 / exp_p).sum())
    dof = max(len(exp_p) - 1, 1)
    return stat <= chi2.ppf(1 - alpha, dof), stat, dof


def test_node2vec_second_order_distribution_chi_square():
    """North-star statistical gate: the GPU's second-order Node2Vec
    transitions follow the exact fp64 probabilities (the reference's
    node2vec_bruteforce, stats.py:142-164, restated here)."""
    g = rmat.rmat_graph(12)
    deg = np.diff(g.offsets)
    s0 = int(np.argsort(deg)[-40])            # a mid-size hub as the start
    n = 400_000
    app = fw.AppConfig(app="node2vec", length=2, a=2.0, b=0.5)
    seq, ln, _ = _run(g, np.full(n, s0, np.int64), app, fw.EngineConfig(replay=True), 123)
    ok = ln == 2
    first, second = seq[ok, 0].astype(np.int64), seq[ok, 1].astype(np.int64)
    checked = 0
    vs, cnt = np.unique(first, return_counts=True)
    for v in vs[np.argsort(cnt)[::-1][:6]]:   # the six most visited first hops
        sel = first == v
        if sel.sum() < 3_000:
            continue
        lo, hi = int(g.offsets[v]), int(g.offsets[v + 1])
        prev_set = set(g.targets[g.offsets[s0]:g.offsets[s0 + 1]].tolist())
        w = []
        for e in range(lo, hi):
            u = int(g.targets[e])
            base = 0.5 if u == s0 else (1.0 if u in prev_set else 2.0)
            w.append(base * float(g.weights[e]))
        w = np.array(w)
        probs = w / w.sum()
        # picks are targets; map them to edge slots (duplicates share mass)
        tg = g.targets[lo:hi].astype(np.int64)
        uniq, inv = np.unique(tg, return_inverse=True)
        p_u = np.bincount(inv, weights=probs, minlength=len(uniq))
        idx = np.searchsorted(uniq, second[sel])
        counts = np.bincount(idx, minlength=len(uniq)).astype(np.float64)
        passed, stat, dof = _chi2_pass(counts, p_u)
        assert passed, (int(v), stat, dof)
        checked += 1
    assert checked >= 3


def test_deepwalk_one_step_distribution_chi_square():
    g = rmat.rmat_graph(12)
    s0 = int(np.argmax(np.diff(g.offsets)))
    n = 300_000
    seq, ln, _ = _run(g, np.full(n, s0, np.int64), fw.AppConfig(app="deepwalk", length=1),
                      fw.EngineConfig(replay=True), 7)
    lo, hi = int(g.offsets[s0]), int(g.offsets[s0 + 1])
    w = g.weights[lo:hi].astype(np.float64)
    tg = g.targets[lo:hi].astype(np.int64)
    uniq, inv = np.unique(tg, return_inverse=True)
    p_u = np.bincount(inv, weights=w / w.sum(), minlength=len(uniq))
    counts = np.bincount(np.searchsorted(uniq, seq[:, 0].astype(np.int64)),
                         minlength=len(uniq)).astype(np.float64)
    passed, stat, dof = _chi2_pass(counts, p_u)
    assert passed, (stat, dof)


def test_overlapped_d2h_pieces_bit_exact(s16):
    """fw_walk copies the result back in 16 pieces while the walk runs (each
    piece waits on the kernel's per-piece completion counter); the host
    arrays must equal the oracle's, bit for bit."""
    from paper_2404_08364_b200 import _lib, engine
    g = s16
    starts = np.arange(g.vertex_count, dtype=np.int64)
    app_cfg = fw.AppConfig(app="node2vec", length=40, a=2.0, b=0.5)
    eng_cfg = fw.EngineConfig(replay=True)
    app, eng, _schema = engine._fw_structs(app_cfg, eng_cfg)
    sess = engine._Session(g, eng_cfg)
    try:
        seq = np.full(len(starts) * app_cfg.length, 7, np.uint32)
        ln = np.full(len(starts), 7, np.uint32)
        st = _lib.FwStats()
        lib = _lib.load()
        rc = lib.fw_walk(sess.handles[0].ptr, starts.ctypes.data, len(starts), 0,
                         engine._ctypes_ref(app), engine._ctypes_ref(eng), 5,
                         seq.ctypes.data, ln.ctypes.data, engine._ctypes_ref(st))
        _lib.check(rc)
    finally:
        sess.close()
    assert st.d2h_pieces == 16 and st.kernel_launches == 1
    oseq, oln, _ = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts,
                               app="node2vec", length=40, a=2.0, b=0.5, seed=5)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq.reshape(len(starts), -1), oseq)


def _clustered_multigraph(seed=11):
    """Hubs whose neighbour lists are long contiguous id ranges with repeated
    entries (multi-edges), overlapping between hubs, plus random edges: skewed
    bucket maps, duplicate keys across 256-slot window boundaries, full
    groups (continuation probes), window advances and the bsearch path."""
    rs = np.random.default_rng(seed)
    V = 8000
    src, dst = [], []
    for h in range(12):
        lo = 400 * h + 20
        nb = np.arange(lo, lo + 2500 + 300 * (h % 4))
        rep = rs.integers(1, 4, len(nb))          # 1-3 copies of each neighbour
        nb = np.repeat(nb, rep)
        src.append(np.full(len(nb), h)); dst.append(nb)
    m = 30000
    src.append(rs.integers(0, V, m)); dst.append(rs.integers(0, V, m))
    s = np.concatenate(src); d = np.concatenate(dst)
    s, d = np.concatenate([s, d]), np.concatenate([d, s])   # symmetrize
    order = np.lexsort((d, s))
    s, d = s[order], d[order]
    off = np.zeros(V + 1, np.int64)
    np.add.at(off, s + 1, 1)
    off = np.cumsum(off)
    w = rs.uniform(1.0, 5.0, len(d)).astype(np.float32)
    return fw.Graph(V, len(d), off, d.astype(np.uint32), w, None)


@pytest.mark.parametrize("eng", [dict(), dict(k_small=4, k_big=8, degree_threshold=6),
                                 dict(k_small=32, k_big=256, degree_threshold=64)])
def test_node2vec_clustered_multigraph_matches_oracle(eng):
    g = _clustered_multigraph()
    starts = np.concatenate([np.arange(g.vertex_count, dtype=np.int64),
                             np.repeat(np.arange(12, dtype=np.int64), 200)])
    app = dict(app="node2vec", length=24, a=2.0, b=0.5)
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True, **eng), 4)
    kw = dict(app)
    kw.update({k: v for k, v in eng.items()})
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, None, starts, seed=4, **kw)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()


def _n2v_weight_sets(n, rs):
    return {
        "u15": rs.uniform(1.0, 5.0, n).astype(np.float32),  # integer tile sums, G = -24
        # small dyadic weights: G = -41, still integer sums (2^41 scale)
        "dyadic": (rs.integers(1, 1 << 20, n).astype(np.float64) * 2.0 ** -40).astype(np.float32),
        # 2^-10 .. 2^25: a lane's scaled sum would overflow u32 -> fp64 tile scan
        "wide": np.where(rs.random(n) < 0.5, 2.0 ** -10, 2.0 ** 25).astype(np.float32),
        "unweighted": None,
    }


@pytest.mark.parametrize("iscan", ["1", "0"])
@pytest.mark.parametrize("wset", ["u15", "dyadic", "wide", "unweighted"])
@pytest.mark.parametrize("ab", [(2.0, 0.5), (0.25, 1.0)])
def test_node2vec_integer_tile_sums_match_oracle(s16, monkeypatch, iscan, wset, ab):
    """Node2Vec's integer tile sums (FW_ISCAN, on when every app weight is a
    multiple of 2^G and a lane's scaled sum fits a u32) and the fp64 tile
    scan give the oracle's paths for weight sets on both sides of the
    eligibility test."""
    monkeypatch.setenv("FW_ISCAN", iscan)
    rs = np.random.default_rng(17)
    w = _n2v_weight_sets(s16.edge_count, rs)[wset]
    g = fw.Graph(s16.vertex_count, s16.edge_count, s16.offsets, s16.targets,
                 w if w is not None else np.ones(s16.edge_count, np.float32), None)
    starts = rs.integers(0, g.vertex_count, 12000).astype(np.int64)
    app = dict(app="node2vec", length=20, a=ab[0], b=ab[1], weighted=w is not None)
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True), 9)
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, None, starts, seed=9, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()


@pytest.mark.parametrize("app", [dict(app="deepwalk", length=40),
                                 dict(app="ppr", length=40, stop_prob=0.2),
                                 dict(app="metapath", length=5, schema=(0, 1, 2, 3, 4))])
def test_rmat_s16_dprs_sampler_matches_oracle(s16, app):
    """The first-order apps under sampler="dprs" (dprs_warp_exact with its
    accept prefilter; hub steps use k = 256) against the oracle."""
    g = s16
    rs = np.random.default_rng(5)
    starts = np.concatenate([rs.integers(0, g.vertex_count, 16000),
                             np.full(500, g.max_degree_vertex())]).astype(np.int64)
    eng = fw.EngineConfig(replay=True, sampler="dprs")
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), eng, 3)
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, seed=3,
                                 sampler="dprs", **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
