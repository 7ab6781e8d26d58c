"""Certified summation (walk mode 2): DPRS and ZPRS over weights whose fp64
partial sums round (log-normal, non-dyadic), with tree-order scans and
certified accept tests instead of the reference's sequential sums
(_kernels.py:404-424, 436-457).  Paths must equal the reference's bit for bit, both on
the fast path and when an ambiguous accept test re-runs the step in order
(forced here by widening the ambiguity band with FW_CERT_SLACK)."""

import os

import numpy as np
import pytest

import oracle
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import rmat
from paper_2404_08364_b200.graph import synthesize_weights

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")


def _run(g, starts, app_cfg, eng_cfg, seed=0):
    seqs, lens = [], []

    def sink(b):
        seqs.append(b.sequences.copy())
        lens.append(b.lengths.copy())

    st = fw.run(g, starts, app_cfg, eng_cfg, seed=seed, sink=sink)
    return np.concatenate(seqs), np.concatenate(lens), st


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *exc):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("slack", [None, "44"])
@pytest.mark.parametrize("name", ["n2v_lognormal", "dw_lognormal_dprs"])
def test_lognormal_goldens_certified(golden, name, slack):
    case = golden.cases[name]
    off, tgt, w, lab = golden.graph(case["graph"])
    g = fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)
    app = dict(case["app"])
    eng = fw.EngineConfig(replay=True, **case["eng"])
    # the golden graphs are small enough that every sum is exact: force mode 2
    env = {"FW_FORCE_CERT": "1", **({"FW_CERT_SLACK": slack} if slack else {})}
    with _env(**env):
        seq, ln, st = _run(g, golden.starts(name), fw.AppConfig(**app), eng, case["seed"])
    want_seq, want_len, want_stats = golden.expected(name)
    assert st.summation == "certified"
    np.testing.assert_array_equal(ln, want_len)
    np.testing.assert_array_equal(seq, want_seq)
    assert [getattr(st, f) for f in STAT_NAMES] == want_stats.tolist()


@pytest.fixture(scope="module")
def s16_lognormal():
    return synthesize_weights(rmat.rmat_graph(16), 2, "lognormal")


@pytest.mark.parametrize("slack", [None, "40"])
@pytest.mark.parametrize("app,sampler", [
    (dict(app="node2vec", length=80, a=2.0, b=0.5), "auto"),
    (dict(app="node2vec", length=40, a=3.0, b=0.7), "auto"),  # fp64 factors
    (dict(app="deepwalk", length=80), "dprs"),
    (dict(app="ppr", length=80, stop_prob=0.2), "dprs"),
    (dict(app="deepwalk", length=80), "auto"),  # ZPRS
    (dict(app="ppr", length=80, stop_prob=0.2), "auto"),
    (dict(app="metapath", length=5, schema=(0, 1, 2, 3, 4)), "auto"),
    (dict(app="node2vec", length=40, a=2.0, b=0.5), "zprs"),
    (dict(app="node2vec", length=40, a=3.0, b=0.7, weighted=False), "auto"),
])
def test_rmat_s16_lognormal_matches_oracle(s16_lognormal, app, sampler, slack):
    g = s16_lognormal
    starts = np.arange(g.vertex_count, dtype=np.int64)
    if slack:  # the forced re-runs are slow: a subset
        starts = starts[::8].copy()
    eng = fw.EngineConfig(replay=True, sampler=sampler)
    with _env(FW_FORCE_CERT="1", **({"FW_CERT_SLACK": slack} if slack else {})):
        seq, ln, st = _run(g, starts, fw.AppConfig(**app), eng)
    assert st.summation == "certified"
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts,
                                 sampler=sampler, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()


def test_certified_equals_ordered_kernels(s16_lognormal):
    """FW_CERT=0 keeps the ordered kernels (the A/B baseline): same paths."""
    g = s16_lognormal
    starts = np.arange(0, g.vertex_count, 4, dtype=np.int64)
    app = fw.AppConfig(app="node2vec", length=80, a=2.0, b=0.5)
    with _env(FW_FORCE_CERT="1"):
        seq_c, ln_c, st_c = _run(g, starts, app, fw.EngineConfig(replay=True))
    with _env(FW_CERT="0", FW_FORCE_CERT="1"):
        seq_o, ln_o, st_o = _run(g, starts, app, fw.EngineConfig(replay=True))
    assert st_c.summation == "certified" and st_o.summation == "sequential"
    with _env(FW_CERT="0"):  # the ordered kernels are the reference's order
        seq_s, _, _ = _run(g, starts, app, fw.EngineConfig(replay=True, order="sequential"))
    np.testing.assert_array_equal(seq_s, seq_o)
    np.testing.assert_array_equal(ln_c, ln_o)
    np.testing.assert_array_equal(seq_c, seq_o)


def test_zprs_hub_groups_certified(s16_lognormal):
    """k = 256 hub steps (8 lane groups, pass 2 from the top group down) and
    PPR's 8-element batches under certification, with forced re-runs."""
    g = s16_lognormal
    hub = g.max_degree_vertex()
    starts = np.full(4096, hub, np.int64)
    for slack in (None, "40"):
        for app in (dict(app="deepwalk", length=20), dict(app="ppr", length=80, stop_prob=0.2)):
            with _env(FW_FORCE_CERT="1", **({"FW_CERT_SLACK": slack} if slack else {})):
                seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True))
            assert st.summation == "certified"
            oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, **app)
            np.testing.assert_array_equal(ln, oln)
            np.testing.assert_array_equal(seq, oseq)
            assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()


def test_unweighted_non_dyadic_factors_select_certified():
    """Unweighted Node2Vec with a = 3, b = 0.7 on a weighted graph: 1/3 and
    1/0.7 make the sums round, so DPRS runs certified (and ignores the
    graph's weights, apps.py weighted=False)."""
    g = rmat.rmat_graph(14)
    starts = np.arange(g.vertex_count, dtype=np.int64)
    app = dict(app="node2vec", length=40, a=3.0, b=0.7, weighted=False)
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True))
    assert st.summation == "certified"
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)


def test_wide_lognormal_selects_certified_on_its_own():
    """Weights spanning ~2^40 (log-normal sigma 4): the exact-order predicate
    fails, so DPRS runs certified without any override."""
    g = synthesize_weights(rmat.rmat_graph(14), 5, "lognormal", sigma=4.0)
    starts = np.arange(g.vertex_count, dtype=np.int64)
    app = dict(app="node2vec", length=40, a=2.0, b=0.5)
    seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True))
    assert st.summation == "certified"
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()


def _golden_names():
    from conftest import Golden
    return sorted(Golden().cases)


@pytest.mark.parametrize("name", _golden_names())
def test_every_golden_case_in_certified_mode(golden, name):
    """Mode 2 forced on all 27 reference goldens: odd and tiny lane widths
    (k = 3..1000, which take the in-order re-run), d_t variants, stars, PPR
    and MetaPath, unweighted runs, the 2^63+5 seed."""
    case = golden.cases[name]
    off, tgt, w, lab = golden.graph(case["graph"])
    g = fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)
    app = dict(case["app"])
    if "schema" in app:
        app["schema"] = tuple(app["schema"])
    eng = fw.EngineConfig(replay=True, **case["eng"])
    with _env(FW_FORCE_CERT="1"):
        seq, ln, st = _run(g, golden.starts(name), fw.AppConfig(**app), eng, case["seed"])
    want_seq, want_len, want_stats = golden.expected(name)
    assert st.summation == "certified"
    np.testing.assert_array_equal(ln, want_len)
    np.testing.assert_array_equal(seq, want_seq)
    assert [getattr(st, f) for f in STAT_NAMES] == want_stats.tolist()


@pytest.mark.parametrize("wbig,wlo,whi", [(5.0e8, 0.9, 1.1), (2.0e8, 0.28, 0.32),
                                           (2.0e8, 0.26, 0.4), (1.0e9, 0.9, 1.1)])
def test_quantized_sums_with_tiny_scaled_weights(wbig, wlo, whi):
    """One huge edge weight puts every other scaled weight near 0.5-1 units of
    the quantized integer sums, so the integer carry overstates the exact one
    by up to 2x: the prefilter must still never reject an element the
    reference accepts (its bound uses carry - 0.5 per element)."""
    g = rmat.rmat_graph(12)
    w = np.random.default_rng(9).uniform(wlo, whi, g.edge_count).astype(np.float32)
    w[np.argmax(np.diff(g.offsets))] = np.float32(wbig)  # one edge somewhere
    g = fw.Graph(g.vertex_count, g.edge_count, g.offsets, g.targets, w, g.labels)
    starts = np.arange(g.vertex_count, dtype=np.int64)
    app = dict(app="node2vec", length=30, a=2.0, b=0.5)
    with _env(FW_FORCE_CERT="1"):
        seq, ln, st = _run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True))
    assert st.summation == "certified"
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts, **app)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
