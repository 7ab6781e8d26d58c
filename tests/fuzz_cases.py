"""Seeded random walk configurations shared by the GPU fuzz test, the oracle
check and tests/golden/gen_fuzz.py (which ran the reference on them): small
skewed edge lists (isolated vertices, self-loops, duplicates, optional
symmetrisation), every app, random lengths / stop probabilities / schemas /
(a, b), lane widths and degree thresholds, both samplers, uniform / integer /
log-normal / zero-heavy / one-huge-weight weights, seeds up to 2^63."""

import numpy as np

N_CASES = 200


def case(seed):
    rs = np.random.default_rng(1000 + seed)
    V = int(rs.integers(1, 400))
    m = int(rs.integers(0, 6000))
    hub = rs.random(m) < 0.3
    src = np.where(hub, rs.integers(0, max(1, V // 20), m), rs.integers(0, V, m))
    dst = rs.integers(0, V, m)
    if rs.random() < 0.5:  # symmetrise (the R-MAT workload's shape)
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    src, dst = src.astype(np.uint32), dst.astype(np.uint32)
    kind = rs.integers(0, 5)
    E = len(src)
    if kind == 0:
        w = rs.uniform(1.0, 5.0, E)
    elif kind == 1:
        w = rs.integers(0, 4, E).astype(np.float64)  # integers, zeros included
    elif kind == 2:
        w = rs.lognormal(0.0, 1.5, E)
    elif kind == 3:
        w = np.where(rs.random(E) < 0.2, 0.0, rs.random(E))
    else:  # one huge weight: the others sit near the quantized sums' resolution
        w = rs.uniform(0.2, 0.7, E)
        if E:
            w[int(rs.integers(0, E))] = float(rs.choice([1e6, 2e8, 1e9, 3e12]))
    lab = rs.integers(0, 5, E).astype(np.uint8)
    app_name = ["deepwalk", "ppr", "node2vec", "metapath"][seed % 4]
    app = dict(app=app_name, length=int(rs.integers(1, 40)), weighted=bool(rs.random() < 0.8))
    if app_name == "ppr":
        app["stop_prob"] = float(rs.choice([0.05, 0.2, 0.5]))
    if app_name == "node2vec":
        app["a"], app["b"] = [(2.0, 0.5), (1.0, 1.0), (3.0, 0.7), (0.25, 4.0)][int(rs.integers(0, 4))]
    if app_name == "metapath":
        app["schema"] = tuple(int(x) for x in rs.integers(0, 5, int(rs.integers(1, 6))))
    k_small = int(rs.choice([1, 2, 3, 4, 8, 16, 32, 33]))
    k_big = int(max(k_small, rs.choice([4, 8, 32, 64, 100, 256, 300])))
    eng = dict(k_small=k_small, k_big=k_big, degree_threshold=int(rs.choice([1, 6, 40, 1024])),
               sampler=str(rs.choice(["auto", "dprs", "zprs"])))
    n = int(rs.integers(1, 300))
    starts = rs.integers(0, V, n).astype(np.int64)
    return dict(src=src, dst=dst, w=w.astype(np.float32), lab=lab, V=V, app=app, eng=eng,
                starts=starts, seed=int(rs.integers(0, 2**63)))


def digest(a):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
