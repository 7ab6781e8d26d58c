"""Generate golden graph-ingest vectors by running the REFERENCE itself.

reswalk's build_csr (graph.py:138-169), parse_edge_list (graph.py:90-135) and
save_binary (graph.py:204-222) on a few edge lists chosen for the tie rule
(many duplicate (src, dst) pairs with distinct weights/labels, so the stable
input order of duplicates is visible), isolated vertices, self loops, an
empty list and a star.  Outputs go to tests/golden/ingest.npz; one FWG1 file
written by the reference is stored as tests/golden/ref_graph.fwg.  Runs only
in the build container (it imports reswalk from /root/reference):

    python tests/golden/gen_ingest.py
"""

import os
import sys

import numpy as np

REF = os.environ.get("RESWALK_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from reswalk.graph import (EdgeList, build_csr, parse_edge_list, save_binary,  # noqa: E402
                           star_edge_list)

OUT = os.path.dirname(os.path.abspath(__file__))


def edge_lists():
    rs = np.random.default_rng(2024)
    out = {}
    m = 20000  # 64 vertices: ~5 copies of every (src, dst) pair
    out["dups64"] = (EdgeList(rs.integers(0, 64, m).astype(np.uint32),
                              rs.integers(0, 64, m).astype(np.uint32),
                              rs.uniform(0.5, 3.0, m).astype(np.float32),
                              rs.integers(0, 256, m).astype(np.uint8)), 70)
    m = 100000  # sparse ids up to 2^17 with isolated vertices, skewed sources
    src = (rs.zipf(1.3, m) % (1 << 17)).astype(np.uint32)
    out["zipf17"] = (EdgeList(src, rs.integers(0, 1 << 17, m).astype(np.uint32),
                              rs.uniform(0.0, 9.0, m).astype(np.float32),
                              rs.integers(0, 5, m).astype(np.uint8)), None)
    out["star"] = (star_edge_list(5000), None)
    out["empty"] = (EdgeList(np.zeros(0, np.uint32), np.zeros(0, np.uint32),
                             np.zeros(0, np.float32), np.zeros(0, np.uint8)), 5)
    text = "# c\n3 1 2.5 4\n3 1 1.5 2\n0 0\n% x\n2 3 7 1\n3 0 1 0\n3 1 0.25 9\n"
    out["parsed_undirected"] = (parse_edge_list(text, undirected=True), 6)
    return out


def main():
    arrays = {}
    for name, (el, vc) in edge_lists().items():
        g = build_csr(el, vc)
        arrays[f"in_{name}_src"] = el.src
        arrays[f"in_{name}_dst"] = el.dst
        arrays[f"in_{name}_w"] = el.weight
        arrays[f"in_{name}_lab"] = el.label
        arrays[f"in_{name}_vc"] = np.array(-1 if vc is None else vc, np.int64)
        arrays[f"out_{name}_offsets"] = g.offsets
        arrays[f"out_{name}_targets"] = g.targets
        arrays[f"out_{name}_weights"] = g.weights
        arrays[f"out_{name}_labels"] = g.labels
        if name == "dups64":
            save_binary(g, os.path.join(OUT, "ref_graph.fwg"))
    np.savez_compressed(os.path.join(OUT, "ingest.npz"), **arrays)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
