"""Run the REFERENCE on the seeded fuzz configurations (tests/fuzz_cases.py)
and record per case the SHA-256 of its sequences and lengths plus the six
RunStats counters (tests/golden/fuzz.json): the oracle (tests/test_oracle.py)
and the CUDA path (tests/test_gpu_fuzz.py) are checked against them.

Runs only in the build container (imports reswalk from /root/reference):

    NUMBA_CACHE_DIR=/tmp/nbc python tests/golden/gen_fuzz.py
"""

import json
import os
import sys

import numpy as np

REF = os.environ.get("RESWALK_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbc")

from reswalk import engine as E  # noqa: E402
from reswalk.apps import AppConfig  # noqa: E402
from reswalk.graph import EdgeList, build_csr  # noqa: E402

import fuzz_cases  # noqa: E402


def main():
    out = []
    for seed in range(fuzz_cases.N_CASES):
        c = fuzz_cases.case(seed)
        g = build_csr(EdgeList(c["src"], c["dst"], c["w"], c["lab"]), c["V"])
        eng = E.EngineConfig(replay=True, workers=2, **c["eng"])
        seqs, lens = [], []

        def sink(b):
            seqs.append(b.sequences.copy())
            lens.append(b.lengths.copy())

        st = E.run(g, c["starts"], AppConfig(**c["app"]), eng, seed=c["seed"], sink=sink)
        seq, ln = np.concatenate(seqs), np.concatenate(lens)
        out.append(dict(seed=seed, seq_sha256=fuzz_cases.digest(seq.astype("<u4")),
                        len_sha256=fuzz_cases.digest(ln.astype("<u4")),
                        stats=[int(st.steps), int(st.edges_scanned), int(st.collectives),
                               int(st.draws), int(st.small_tasks), int(st.large_tasks)],
                        sampled=int(ln.astype(np.int64).sum())))
    with open(os.path.join(HERE, "fuzz.json"), "w") as fh:
        json.dump(dict(generator="tests/golden/gen_fuzz.py",
                       reference="reswalk (/root/reference/pkg), replay mode, workers=2",
                       cases=out), fh, indent=0)
    print(f"{len(out)} cases, {sum(c['sampled'] for c in out)} sampled steps")


if __name__ == "__main__":
    main()
