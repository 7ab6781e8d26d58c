#!/usr/bin/env python
"""North-star evidence run (not a bench line): Node2Vec a=2 b=0.5 L=80 on the
R-MAT scale-27 graph (2^27 vertices, 2^31 CSR entries), one query per vertex,
on one B200.

  1. the whole job as one walk launch (134M queries, 43 GB of paths in HBM),
     then the GPU validate_walks over every path (_kernels.py:486-546);
  2. the same qid range cut into the 8 contiguous partitions an 8-GPU run
     would give each rank (bench.py --scaling strong), each timed alone: an
     8-GPU job has no communication on the walk path, so its walk time is the
     slowest partition's.

Prints one JSON line.  Device time by CUDA events on the launching stream.
"""

import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2404_08364_b200 as fw  # noqa: E402
from paper_2404_08364_b200 import _lib, rmat  # noqa: E402
from paper_2404_08364_b200.engine import _fw_structs  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    parts = 8
    lib = _lib.load()
    dev = torch.device("cuda:0")
    t0 = time.perf_counter()
    dg = rmat.rmat_graph_device(scale, labels=False, device=0)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    V = dg.vertex_count
    h = dg.handle(0).ptr
    L = 80
    app = fw.AppConfig(app="node2vec", length=L, a=2.0, b=0.5)
    a_s, e_s, _ = _fw_structs(app, fw.EngineConfig(replay=True))
    starts = torch.arange(V, dtype=torch.int64, device=dev)
    seq = torch.empty(V * L, dtype=torch.int32, device=dev)
    lens = torch.empty(V, dtype=torch.int32, device=dev)
    stats = torch.zeros(10, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def walk(lo, hi):
        stats.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(lib.fw_walk_device(h, starts[lo:].data_ptr(), hi - lo, lo, ctypes.byref(a_s),
                                      ctypes.byref(e_s), 0, seq[lo * L:].data_ptr(),
                                      lens[lo:].data_ptr(), stats.data_ptr(), stream.cuda_stream))
        e1.record(stream)
        torch.cuda.synchronize()
        st = stats.cpu().tolist()
        return e0.elapsed_time(e1), st

    # 1. the whole job in one launch, then validate every path on the GPU
    ms, st = walk(0, V)
    sampled, alg = st[6], st[7]
    bad = torch.zeros(1, dtype=torch.int64, device=dev)
    tv = time.perf_counter()
    _lib.check(lib.fw_validate_device(h, starts.data_ptr(), V, seq.data_ptr(), lens.data_ptr(),
                                      L, None, 0, bad.data_ptr(), stream.cuda_stream))
    torch.cuda.synchronize()
    val_s = time.perf_counter() - tv
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6505.6
    one = {"queries": V, "ms": ms, "sampled_steps": sampled, "steps_per_s": sampled / (ms / 1e3),
           "alg_bytes": alg, "roofline_frac": alg / (ms / 1e3) / 1e9 / peak,
           "validate_violations": int(bad.item()), "validate_s": val_s}
    # 2. the 8 partitions of an 8-GPU strong-scaling run, one at a time
    part = []
    for r in range(parts):
        lo, hi = r * V // parts, (r + 1) * V // parts
        pms, pst = walk(lo, hi)
        part.append({"rank": r, "queries": hi - lo, "ms": pms, "sampled_steps": pst[6],
                     "alg_bytes": pst[7]})
    slow = max(p["ms"] for p in part)
    tot = sum(p["sampled_steps"] for p in part)
    tot_b = sum(p["alg_bytes"] for p in part)
    print(json.dumps({
        "what": f"Node2Vec a=2 b=0.5 L=80, R-MAT scale-{scale} ef16, one query per vertex, 1 B200",
        "graph": {"vertices": V, "csr_entries": dg.edge_count, "gen_s": gen_s,
                  "max_degree": dg.max_degree()},
        "single_launch": one,
        "partitions_8": part,
        "projected_8gpu": {
            "note": "8 replicas, disjoint qid ranges, no walk-path communication: job time = "
                    "slowest partition (each timed alone on this GPU)",
            "ms": slow, "steps_per_s": tot / (slow / 1e3),
            "roofline_frac_of_8x_peak": tot_b / (slow / 1e3) / 1e9 / (8 * peak),
            "partition_imbalance": slow / (sum(p["ms"] for p in part) / parts)},
        "peak_gbs": peak}))


if __name__ == "__main__":
    main()
