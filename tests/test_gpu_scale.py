"""Bit-exact parity at the BASELINE.json configurations' own scale.

The graphs are the benchmarked ones (R-MAT ef16, built on the device by
``rmat_graph_device`` exactly as bench.py builds them), copied to the host for
the C oracle (a restatement of reswalk ``_kernels.step_pass``,
``_kernels.py:320-483``).  Each block is a run of consecutive *global* query
ids walked through the public API (``run(..., base_qid=...)`` -> ``fw_walk``);
in replay mode a walk is a pure function of its global qid, so a block equals
the same rows of the full benchmark run.  Paths, lengths and all six RunStats
counters must match bit for bit.

  config 2  Node2Vec a=2 b=0.5 L80, s22: first / random interior / last qid
            blocks (start = qid) and a block starting every query at the hub;
            chi-square of the second-order transition out of the hub
  config 3  MetaPath schema (0..4) L5, labelled s24: all-vertex blocks
  config 4  PPR stop 0.2 L80, s24: queries starting at the max-degree vertex
  config 5  Node2Vec s27 (2^31 CSR entries): interior and hub blocks
"""

import os

import numpy as np
import pytest

import oracle
from conftest import chi2_pass
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import rmat

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")
THREADS = os.cpu_count() or 1


def _gpu(dg, starts, app_cfg, base_qid, seed=0, eng=None):
    seqs, lens = [], []

    def sink(b):
        seqs.append(b.sequences.copy())
        lens.append(b.lengths.copy())

    st = fw.run(dg, starts, app_cfg, eng or fw.EngineConfig(replay=True), seed=seed, sink=sink,
                base_qid=base_qid)
    return np.concatenate(seqs), np.concatenate(lens), st


def _check_block(dg, host, starts, app_cfg, base_qid, seed=0):
    seq, ln, st = _gpu(dg, starts, app_cfg, base_qid, seed)
    kw = dict(app=app_cfg.app, length=app_cfg.length, stop_prob=app_cfg.stop_prob, a=app_cfg.a,
              b=app_cfg.b, schema=tuple(app_cfg.schema), weighted=app_cfg.weighted)
    oseq, oln, ost = oracle.walk(host.offsets, host.targets, host.weights, host.labels, starts,
                                 base_qid=base_qid, seed=seed, threads=THREADS, **kw)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
    assert st.sampled_steps == int(oln.astype(np.int64).sum())
    assert st.exact_order
    return seq, ln, st


# ---------------------------------------------------------------------------
# config 2: Node2Vec s22
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def s22():
    dg = rmat.rmat_graph_device(22, labels=False)
    host = dg.to_host()
    yield dg, host
    dg.close()


N2V = fw.AppConfig(app="node2vec", length=80, a=2.0, b=0.5)


@pytest.mark.parametrize("block", ["first", "interior", "last", "hub"])
def test_s22_node2vec_blocks(s22, block):
    dg, host = s22
    V, nq = host.vertex_count, 1024
    if block == "first":
        base = 0
    elif block == "interior":
        base = int(np.random.default_rng(22).integers(nq, V - 2 * nq))
    elif block == "last":
        base = V - nq
    else:
        base = 1_234_567
    starts = (np.full(nq, host.max_degree_vertex(), np.int64) if block == "hub"
              else np.arange(base, base + nq, dtype=np.int64))
    _seq, ln, st = _check_block(dg, host, starts, N2V, base)
    assert st.sampled_steps > 0
    if block == "hub":
        assert st.large_tasks >= nq and st.edges_scanned > nq * host.max_degree()


@pytest.mark.parametrize("block", ["interior", "hub"])
def test_s22_node2vec_lognormal_certified_blocks(s22, block):
    """The certified mode at the benchmark's scale: the s22 graph with
    log-normal weights (bench.py --weights lognormal; sums round, so the walk
    runs tree-order integer sums with certified accept tests), against the
    oracle's sequential sums on the same qids."""
    import torch
    dg0, host0 = s22
    E = host0.edge_count
    w = np.random.default_rng(2).lognormal(0.0, 1.0, E).astype(np.float32)
    wd = torch.empty(E + 4, dtype=torch.float32, device="cuda")[:E]
    wd.copy_(torch.from_numpy(w))
    from paper_2404_08364_b200.engine import DeviceGraph
    dg = DeviceGraph(host0.vertex_count, E, dg0.offsets, dg0.targets, wd, None, device=0)
    host = fw.Graph(host0.vertex_count, E, host0.offsets, host0.targets, w, None)
    V, nq = host.vertex_count, 1024
    base = 3_000_000 if block == "interior" else 777_777
    starts = (np.full(nq, host.max_degree_vertex(), np.int64) if block == "hub"
              else np.arange(base, base + nq, dtype=np.int64))
    seq, ln, st = _gpu(dg, starts, N2V, base)
    assert st.summation == "certified"
    oseq, oln, ost = oracle.walk(host.offsets, host.targets, host.weights, None, starts,
                                 app="node2vec", length=80, a=2.0, b=0.5, base_qid=base,
                                 threads=THREADS)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
    dg.close()


def test_s22_node2vec_out_of_hub_chi_square(s22):
    """Second-order transitions out of the s22 hub: start at s0 (a neighbour
    of the hub with a sizable N(s0)); conditioned on the first hop being the
    hub, the second hop must follow f(u) * w(hub, u) with f = 1/a for u == s0,
    1 for u in N(s0), 1/b otherwise (the reference's node2vec_bruteforce,
    stats.py:142-164).  The first hop out of s0 is checked too."""
    dg, host = s22
    off, tgt, w = host.offsets, host.targets, host.weights
    hub = host.max_degree_vertex()
    nb = tgt[off[hub]:off[hub + 1]].astype(np.int64)
    cand = np.unique(nb)
    deg = off[cand + 1] - off[cand]
    cand = cand[(deg >= 200) & (deg <= 4000)]
    best, p_best = None, 0.0
    for v in cand[:4000]:
        lo, hi = int(off[v]), int(off[v + 1])
        ww = w[lo:hi].astype(np.float64)
        p = ww[tgt[lo:hi] == hub].sum() / ww.sum()
        if p > p_best:
            best, p_best = int(v), p
    assert best is not None
    n = int(min(150_000_000, np.ceil(500_000 / p_best)))
    app = fw.AppConfig(app="node2vec", length=2, a=2.0, b=0.5)
    seq, ln, _ = _gpu(dg, np.full(n, best, np.int64), app, 0, seed=31)
    # first hop out of s0 (first-order: prev = -1)
    lo, hi = int(off[best]), int(off[best + 1])
    t0 = tgt[lo:hi].astype(np.int64)
    uniq, inv = np.unique(t0, return_inverse=True)
    p1 = np.bincount(inv, weights=w[lo:hi].astype(np.float64), minlength=len(uniq))
    c1 = np.bincount(np.searchsorted(uniq, seq[:, 0].astype(np.int64)), minlength=len(uniq))
    ok, stat, dof = chi2_pass(c1, p1 / p1.sum())
    assert ok, ("first hop", stat, dof)
    # second hop out of the hub, conditioned on first == hub
    sel = (seq[:, 0] == hub) & (ln == 2)
    second = seq[sel, 1].astype(np.int64)
    assert len(second) > 300_000
    nprev = set(t0.tolist())
    lo, hi = int(off[hub]), int(off[hub + 1])
    th = tgt[lo:hi].astype(np.int64)
    f = np.where(th == best, 0.5, np.where(np.isin(th, list(nprev)), 1.0, 2.0))
    pw = f * w[lo:hi].astype(np.float64)
    uniq, inv = np.unique(th, return_inverse=True)
    p2 = np.bincount(inv, weights=pw, minlength=len(uniq))
    c2 = np.bincount(np.searchsorted(uniq, second), minlength=len(uniq))
    ok, stat, dof = chi2_pass(c2, p2 / p2.sum())
    assert ok, ("second hop out of the hub", stat, dof)


# ---------------------------------------------------------------------------
# configs 3 and 4: labelled s24
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def s24():
    dg = rmat.rmat_graph_device(24, labels=True)
    host = dg.to_host()
    yield dg, host
    dg.close()


@pytest.mark.parametrize("block", ["first", "last"])
def test_s24_metapath_all_vertex_blocks(s24, block):
    dg, host = s24
    V = host.vertex_count
    nq = 1 << 18 if block == "first" else 1 << 16
    base = 0 if block == "first" else V - nq
    app = fw.AppConfig(app="metapath", length=5, schema=(0, 1, 2, 3, 4))
    seq, ln, st = _check_block(dg, host, np.arange(base, base + nq, dtype=np.int64), app, base)
    assert oracle.validate(host.offsets, host.targets, host.labels,
                           np.arange(base, base + nq), seq, ln, (0, 1, 2, 3, 4)) == 0


@pytest.mark.parametrize("base", [0, 9_000_000])
def test_s24_ppr_hub_starts(s24, base):
    dg, host = s24
    nq = 4096
    app = fw.AppConfig(app="ppr", length=80, stop_prob=0.2)
    _seq, _ln, st = _check_block(dg, host, np.full(nq, host.max_degree_vertex(), np.int64),
                                 app, base)
    assert st.draws > 0 and st.large_tasks >= nq // 2


# ---------------------------------------------------------------------------
# config 5: Node2Vec s27 (2^31 CSR entries: int64 offsets, 64-bit edge ids)
# ---------------------------------------------------------------------------
def _s27_resources_ok():
    try:
        import psutil
        import torch
        free, _total = torch.cuda.mem_get_info(0)
        return psutil.virtual_memory().available > 40 << 30 and free > 90 << 30
    except Exception:
        return False


def test_s27_node2vec_blocks():
    if not _s27_resources_ok():
        pytest.skip("s27 needs > 90 GB free HBM and > 40 GB host RAM")
    dg = rmat.rmat_graph_device(27, labels=False)
    try:
        host = dg.to_host()
        assert host.edge_count == 1 << 31
        V = host.vertex_count
        base = int(np.random.default_rng(27).integers(0, V - 4096))
        _check_block(dg, host, np.arange(base, base + 4096, dtype=np.int64), N2V, base)
        _check_block(dg, host, np.full(1024, host.max_degree_vertex(), np.int64), N2V,
                     V - 1024)
    finally:
        dg.close()
