"""Generate golden walk vectors by running the REFERENCE itself.

Runs only in the build container (it imports reswalk from /root/reference);
the outputs are committed as tests/golden/walks.npz + cases.json and are what
the oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_parity.py)
are pinned against on the GPU box, where /root/reference does not exist.

    NUMBA_CACHE_DIR=/tmp/nbc python tests/golden/gen_golden.py
"""

import json
import os
import sys

import numpy as np

REF = os.environ.get("RESWALK_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..")))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbc")

from reswalk import engine as E  # noqa: E402
from reswalk.apps import AppConfig  # noqa: E402
from reswalk.graph import (build_csr, random_edge_list, star_edge_list,  # noqa: E402
                           synthesize_weights)
from reswalk.rng import mix64, stream_base, value_at  # noqa: E402

from paper_2404_08364_b200 import rmat  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def graphs():
    g = {}
    r = rmat.rmat_graph(10)
    g["rmat10"] = (r.offsets, r.targets, r.weights, r.labels)
    # non-dyadic weights: fp64 partial sums round, so summation order matters
    from reswalk.graph import Graph
    rg = Graph(r.vertex_count, r.edge_count, r.offsets, r.targets, r.weights, r.labels)
    ln = synthesize_weights(rg, 7, "lognormal", 0.0, 1.0)
    g["rmat10_lognormal"] = (ln.offsets, ln.targets, ln.weights, ln.labels)
    s = build_csr(star_edge_list(3000), 3001)
    s = synthesize_weights(s, 11, "uniform")
    g["star3000"] = (s.offsets, s.targets, s.weights, None)
    rnd = build_csr(random_edge_list(40, 300, 123), 40)
    w = np.random.default_rng(5).uniform(0.1, 4, rnd.edge_count).astype(np.float32)
    g["rand40"] = (rnd.offsets, rnd.targets, w, None)
    r12 = rmat.rmat_graph(12)
    g["rmat12"] = (r12.offsets, r12.targets, r12.weights, r12.labels)
    return g


def cases(gs):
    V10 = len(gs["rmat10"][0]) - 1
    hub10 = int(np.argmax(np.diff(gs["rmat10"][0])))
    allv = list(range(V10))
    c = []

    def add(name, graph, starts, app, eng=None, seed=0):
        c.append(dict(name=name, graph=graph, starts=[int(x) for x in starts], app=app,
                      eng=eng or {}, seed=seed))

    add("dw_l20", "rmat10", allv, dict(app="deepwalk", length=20))
    add("dw_l20_dprs", "rmat10", allv, dict(app="deepwalk", length=20), dict(sampler="dprs"))
    add("dw_unweighted", "rmat10", allv, dict(app="deepwalk", length=12, weighted=False))
    add("n2v_l20", "rmat10", allv, dict(app="node2vec", length=20, a=2.0, b=0.5))
    add("n2v_l20_zprs", "rmat10", allv, dict(app="node2vec", length=20), dict(sampler="zprs"))
    add("n2v_unweighted", "rmat10", allv, dict(app="node2vec", length=12, weighted=False))
    add("n2v_a3_b07", "rmat10", allv, dict(app="node2vec", length=16, a=3.0, b=0.7))
    add("ppr_hub", "rmat10", [hub10] * 400, dict(app="ppr", length=20, stop_prob=0.2))
    add("ppr_all", "rmat10", allv, dict(app="ppr", length=30, stop_prob=0.3),
        dict(sampler="dprs"))
    add("mp_schema5", "rmat10", allv, dict(app="metapath", length=80, schema=[0, 1, 2, 3, 4]))
    add("mp_schema3_unw", "rmat10", allv,
        dict(app="metapath", length=2, schema=[1, 1, 0], weighted=False), dict(sampler="dprs"))
    add("dw_small_k", "rmat10", allv[:300], dict(app="deepwalk", length=10),
        dict(k_small=4, k_big=8, degree_threshold=6))
    add("dw_small_k_dprs", "rmat10", allv[:300], dict(app="deepwalk", length=10),
        dict(k_small=4, k_big=8, degree_threshold=6, sampler="dprs"))
    add("n2v_small_k", "rmat10", allv[:300], dict(app="node2vec", length=10),
        dict(k_small=4, k_big=8, degree_threshold=6))
    add("n2v_odd_k", "rmat10", allv[:300], dict(app="node2vec", length=10),
        dict(k_small=3, k_big=1000, degree_threshold=50))
    add("dw_odd_k_zprs", "rmat10", allv[:300], dict(app="deepwalk", length=10),
        dict(k_small=5, k_big=77, degree_threshold=40))
    add("dw_lognormal", "rmat10_lognormal", allv, dict(app="deepwalk", length=16))
    add("dw_lognormal_dprs", "rmat10_lognormal", allv, dict(app="deepwalk", length=16),
        dict(sampler="dprs"))
    add("n2v_lognormal", "rmat10_lognormal", allv, dict(app="node2vec", length=16))
    add("star_dw", "star3000", [0] * 40 + list(range(1, 41)), dict(app="deepwalk", length=6))
    add("star_dw_dprs", "star3000", [0] * 40 + list(range(1, 41)),
        dict(app="deepwalk", length=6), dict(sampler="dprs"))
    add("star_n2v", "star3000", [0] * 40 + list(range(1, 41)), dict(app="node2vec", length=6))
    add("star_ppr", "star3000", [0] * 60, dict(app="ppr", length=10, stop_prob=0.2))
    add("rand40_dw", "rand40", list(range(40)) * 3, dict(app="deepwalk", length=8),
        dict(k_small=4, k_big=8, degree_threshold=6))
    add("dw_bigseed", "rmat10", allv[:500], dict(app="deepwalk", length=10), seed=2**63 + 5)
    add("dw_batched", "rmat10", allv, dict(app="deepwalk", length=8),
        dict(memory_budget=2 * 9 * 4 * 300, graph_bytes=0))
    add("n2v_rmat12", "rmat12", list(range(0, 4096, 2)), dict(app="node2vec", length=24))
    return c


def run_case(gs, case):
    from reswalk.graph import Graph
    off, tgt, w, lab = gs[case["graph"]]
    g = Graph(len(off) - 1, len(tgt), off, tgt, w, lab)
    app = dict(case["app"])
    if "schema" in app:
        app["schema"] = tuple(app["schema"])
    app_cfg = AppConfig(**app)
    eng_cfg = E.EngineConfig(replay=True, workers=2, **case["eng"])
    starts = np.asarray(case["starts"], np.int64)
    seqs, lens = [], []

    def sink(b):
        seqs.append(b.sequences.copy())
        lens.append(b.lengths.copy())

    st = E.run(g, starts, app_cfg, eng_cfg, seed=case["seed"], sink=sink)
    stats = [st.steps, st.edges_scanned, st.collectives, st.draws, st.small_tasks, st.large_tasks]
    return np.concatenate(seqs), np.concatenate(lens), np.asarray(stats, np.int64)


def kats():
    rows = []
    for key, sid, ctr in [(7, 0, 0), (7, 0, 1), (7, 1, 0), (0, 1 << 63, 0),
                          (42, (1 << 63) | (5 << 30) | (3 << 10) | 1023, 0),
                          (2**63, 1 << 40, 5), (123, 99, 68), (2**64 - 1, 2**64 - 1, 2**40)]:
        base = stream_base(key, sid)
        z = mix64((base + ctr * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
        rows.append(dict(key=str(key), sid=str(sid), ctr=str(ctr), base=str(base), z=str(z),
                         u01=value_at(key, sid, ctr)))
    return rows


def trial_cases():
    """Sampler trial kernels (_kernels.py:84-277) through trials.run_trials."""
    from reswalk import _kernels as K
    from reswalk.samplers import WeightOracle, alias_build
    rng = np.random.default_rng(77)
    out, arrays = [], {}
    vecs = {
        "u12": rng.uniform(0, 5, 12),
        "z23": np.where(rng.random(23) < 0.35, 0.0, rng.uniform(0, 5, 23)),
        "ln300": rng.lognormal(0.0, 1.5, 300),
        "one": np.array([2.5]),
        "n1000": rng.uniform(0.1, 4.0, 1000),
    }
    for vname, w in vecs.items():
        arrays[f"t_w_{vname}"] = w
        tab = alias_build(WeightOracle.from_array(w))
        arrays[f"t_aliasprob_{vname}"] = tab.prob
        arrays[f"t_aliasidx_{vname}"] = tab.alias
        for seed in (3, 2**63 + 11):
            key = np.uint64(seed)
            T = 200
            runs = [("seq", 1, K.seq_rs_trials(w, key, T), None),
                    ("its", 1, K.its_trials(w, key, T), None),
                    ("alias", 1, K.alias_trials(tab.prob, tab.alias, key, T), None),
                    ("uniform-control", 1, K.uniform_control_trials(len(w), key, T), None)]
            pr, rd = K.rjs_trials(w, float(w.max()), key, T, 10_000)
            runs.append(("rjs", 1, pr, rd))
            for k in (1, 3, 32, 256):
                pd, cd = K.dprs_trials(w, k, key, T)
                pz, cz = K.zprs_trials(w, k, key, T)
                runs += [("dprs", k, pd, cd), ("zprs", k, pz, cz)]
            for sampler, k, picks, aux in runs:
                name = f"{vname}_{sampler}_{k}_{seed}"
                arrays[f"t_picks_{name}"] = np.asarray(picks)
                if aux is not None:
                    arrays[f"t_aux_{name}"] = np.asarray(aux)
                out.append(dict(name=name, vec=vname, sampler=sampler, k=k, seed=str(seed),
                                trials=T))
    return out, arrays


def main():
    gs = graphs()
    arrays = {}
    for name, (off, tgt, w, lab) in gs.items():
        arrays[f"g_{name}_offsets"] = off
        arrays[f"g_{name}_targets"] = tgt
        arrays[f"g_{name}_weights"] = w
        if lab is not None:
            arrays[f"g_{name}_labels"] = lab
    cs = cases(gs)
    for case in cs:
        seq, ln, st = run_case(gs, case)
        arrays[f"c_{case['name']}_seq"] = seq
        arrays[f"c_{case['name']}_len"] = ln
        arrays[f"c_{case['name']}_stats"] = st
        arrays[f"c_{case['name']}_starts"] = np.asarray(case.pop("starts"), np.int64)
        print(f"{case['name']:20s} n={len(ln):5d} sampled={int(ln.sum()):7d} stats={st.tolist()}")
    tcases, tarrays = trial_cases()
    arrays.update(tarrays)
    np.savez_compressed(os.path.join(OUT, "walks.npz"), **arrays)
    meta = dict(cases=cs, kats=kats(), trials=tcases, generator="tests/golden/gen_golden.py",
                reference="reswalk 0.1.0 (/root/reference/pkg), replay mode, workers=2")
    with open(os.path.join(OUT, "cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
