#!/usr/bin/env python
"""Bit-exactness spot check at the north-star scale (test infrastructure: it
runs the CPU oracle as the checker).  Node2Vec a=2 b=0.5 L=80 on R-MAT
scale-27: the GPU walks blocks of global query ids, the C oracle walks the
same (start, qid) pairs on the host copy of the same CSR, and paths, lengths
and the six RunStats counters must match bit for bit.  Prints one JSON line.
"""

import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2404_08364_b200 as fw  # noqa: E402
from paper_2404_08364_b200 import _lib, rmat  # noqa: E402
from paper_2404_08364_b200.engine import _fw_structs  # noqa: E402


def main():
    scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    per_block = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    lib = _lib.load()
    dev = torch.device("cuda:0")
    dg = rmat.rmat_graph_device(scale, labels=False, device=0)
    V = dg.vertex_count
    t0 = time.perf_counter()
    host = dg.to_host()
    copy_s = time.perf_counter() - t0
    L = 80
    app = fw.AppConfig(app="node2vec", length=L, a=2.0, b=0.5)
    a_s, e_s, _ = _fw_structs(app, fw.EngineConfig(replay=True))
    hub = dg.max_degree_vertex()
    rs = np.random.default_rng(27)
    # blocks of consecutive qids: the start, a random interior block, the end,
    # and a block whose starts are all the hub (qids still distinct)
    firsts = [0, int(rs.integers(per_block, V - 2 * per_block)), V - per_block]
    blocks = [(q, np.arange(q, q + per_block, dtype=np.int64)) for q in firsts]
    blocks.append((int(rs.integers(0, V - per_block)), np.full(per_block, hub, np.int64)))
    out = []
    ok = True
    for q0, st in blocks:
        n = len(st)
        starts = torch.from_numpy(st).to(dev)
        seq = torch.empty(n * L, dtype=torch.int32, device=dev)
        lens = torch.empty(n, dtype=torch.int32, device=dev)
        stats = torch.zeros(10, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev)
        _lib.check(lib.fw_walk_device(dg.handle(0).ptr, starts.data_ptr(), n, q0,
                                      ctypes.byref(a_s), ctypes.byref(e_s), 0, seq.data_ptr(),
                                      lens.data_ptr(), stats.data_ptr(), stream.cuda_stream))
        torch.cuda.synchronize()
        gseq = seq.cpu().numpy().view(np.uint32).reshape(n, L)
        glen = lens.cpu().numpy().view(np.uint32)
        gst = stats.cpu().numpy()[:6].tolist()
        t1 = time.perf_counter()
        oseq, oln, ost = oracle.walk(host.offsets, host.targets, host.weights, None, st,
                                     app="node2vec", length=L, a=2.0, b=0.5, base_qid=q0)
        osec = time.perf_counter() - t1
        same = bool(np.array_equal(gseq, oseq) and np.array_equal(glen, oln) and
                    gst == ost.tolist())
        ok &= same
        out.append({"base_qid": q0, "queries": n, "hub_starts": bool((st == hub).all()),
                    "sampled_steps": int(oln.sum()), "edges_scanned": int(ost[1]),
                    "bit_exact": same, "oracle_s": osec})
    print(json.dumps({"what": f"Node2Vec a=2 b=0.5 L=80, R-MAT scale-{scale}: GPU vs C oracle",
                      "vertices": V, "csr_entries": dg.edge_count, "host_copy_s": copy_s,
                      "blocks": out, "all_bit_exact": ok}))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
