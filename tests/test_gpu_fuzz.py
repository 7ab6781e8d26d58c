"""Seeded random configurations against the oracle: small graphs with
isolated vertices, self-loops, duplicate edges and a skewed degree
distribution; every app; random lane widths and degree thresholds (the
reference's own pins use k = 4/8, d_t = 6, tests/test_kernels.py:100-101);
weights uniform, integer, log-normal or with zeros; all three summation modes.
Paths, lengths and the six RunStats counters must match bit for bit."""

import os

import numpy as np
import pytest

import oracle
import paper_2404_08364_b200 as fw

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")
N_CASES = 200


def _graph(rs):
    V = int(rs.integers(1, 400))
    m = int(rs.integers(0, 6000))
    # skewed endpoints: a few hubs, many low-degree vertices, some isolated
    hub = rs.random(m) < 0.3
    src = np.where(hub, rs.integers(0, max(1, V // 20), m), rs.integers(0, V, m))
    dst = rs.integers(0, V, m)
    if rs.random() < 0.5:  # symmetrise (the R-MAT workload's shape)
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    src, dst = src.astype(np.uint32), dst.astype(np.uint32)
    kind = rs.integers(0, 4)
    E = len(src)
    if kind == 0:
        w = rs.uniform(1.0, 5.0, E)
    elif kind == 1:
        w = rs.integers(0, 4, E).astype(np.float64)  # integers, zeros included
    elif kind == 2:
        w = rs.lognormal(0.0, 1.5, E)
    else:
        w = np.where(rs.random(E) < 0.2, 0.0, rs.random(E))
    lab = rs.integers(0, 5, E).astype(np.uint8)
    el = fw.EdgeList(src, dst, w.astype(np.float32), lab)
    return fw.build_csr(el, V)


def _case(seed):
    rs = np.random.default_rng(1000 + seed)
    g = _graph(rs)
    app_name = ["deepwalk", "ppr", "node2vec", "metapath"][seed % 4]
    app = dict(app=app_name, length=int(rs.integers(1, 40)),
               weighted=bool(rs.random() < 0.8))
    if app_name == "ppr":
        app["stop_prob"] = float(rs.choice([0.05, 0.2, 0.5]))
    if app_name == "node2vec":
        app["a"], app["b"] = [(2.0, 0.5), (1.0, 1.0), (3.0, 0.7), (0.25, 4.0)][int(rs.integers(0, 4))]
    if app_name == "metapath":
        app["schema"] = tuple(int(x) for x in rs.integers(0, 5, int(rs.integers(1, 6))))
        app["length"] = max(app["length"], 1)
    k_small = int(rs.choice([1, 2, 3, 4, 8, 16, 32, 33]))
    k_big = int(max(k_small, rs.choice([4, 8, 32, 64, 100, 256, 300])))
    eng = dict(k_small=k_small, k_big=k_big, degree_threshold=int(rs.choice([1, 6, 40, 1024])),
               sampler=str(rs.choice(["auto", "dprs", "zprs"])))
    n = int(rs.integers(1, 300))
    starts = rs.integers(0, g.vertex_count, n).astype(np.int64)
    return g, app, eng, starts, int(rs.integers(0, 2**63))


def _run(g, starts, app, eng, seed, order, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        seqs, lens = [], []

        def sink(b):
            seqs.append(b.sequences.copy())
            lens.append(b.lengths.copy())

        st = fw.run(g, starts, fw.AppConfig(**app), fw.EngineConfig(replay=True, order=order, **eng),
                    seed=seed, sink=sink)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return np.concatenate(seqs), np.concatenate(lens), st


@pytest.mark.parametrize("mode", ["auto", "sequential", "certified"])
@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_configuration_matches_oracle(seed, mode):
    g, app, eng, starts, wseed = _case(seed)
    kw = dict(app)
    oseq, oln, ost = oracle.walk(g.offsets, g.targets, g.weights, g.labels, starts,
                                 k_small=eng["k_small"], k_big=eng["k_big"],
                                 degree_threshold=eng["degree_threshold"],
                                 sampler=eng["sampler"], seed=wseed, **kw)
    order = "sequential" if mode == "sequential" else "auto"
    env = {"FW_FORCE_CERT": "1"} if mode == "certified" else {}
    seq, ln, st = _run(g, starts, app, eng, wseed, order, env)
    np.testing.assert_array_equal(ln, oln)
    np.testing.assert_array_equal(seq, oseq)
    assert [getattr(st, f) for f in STAT_NAMES] == ost.tolist()
