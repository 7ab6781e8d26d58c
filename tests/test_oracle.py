"""Pins the CPU oracle (oracle/walk_oracle.c) to the reference: golden walk
vectors produced by running reswalk itself, and the RNG known answers."""

import os

import numpy as np
import pytest

import oracle
from conftest import case_kwargs
from paper_2404_08364_b200 import engine, rng


def test_rng_known_answers(golden):
    lib = oracle.oracle_lib()
    for row in golden.kats:
        key, sid, ctr = int(row["key"]), int(row["sid"]), int(row["ctr"])
        base = int(row["base"])
        assert oracle.stream_base(key, sid) == base
        assert lib.fwo_stream_base(key, sid) == base
        assert rng.stream_base(key, sid) == base
        assert oracle.mix64((base + ctr * oracle.GOLDEN) & oracle.oracle.MASK64) == int(row["z"])
        assert lib.fwo_u01(base, ctr) == row["u01"]
        assert rng.value_at(key, sid, ctr) == row["u01"]


def test_rng_survey_appendix_a():
    # SURVEY.md Appendix A, generated from the reference rng.py
    assert rng.mix64(0) == 0
    assert rng.mix64(1) == 0x5692161D100B05E5
    assert rng.stream_base(7, 0) == 0x74B5ABCC66B8BDC1
    assert rng.value_at(7, 0, 0) == 0.065771917505381583
    assert rng.stream_base(0, 1 << 63) == 0x42F83292896BFC97
    assert rng.value_at(42, 0x8000000140000FFF, 0) == 0.97836018574807104
    assert rng.stream_base(2**63, 0x10000000000) == 0xB415F27AB9F3D42E


def _cases():
    from conftest import Golden
    return sorted(Golden().cases)


@pytest.mark.parametrize("name", _cases())
def test_oracle_matches_reference_golden(golden, name):
    case = golden.cases[name]
    off, tgt, w, lab = golden.graph(case["graph"])
    starts = golden.starts(name)
    want_seq, want_len, want_stats = golden.expected(name)
    kw, eng = case_kwargs(case)
    if "memory_budget" in eng:
        # batched run: same global qids, so one unbatched oracle call matches
        size = engine.batch_size(engine.EngineConfig(**eng), kw["length"])
        assert size < len(starts)
    seq, ln, st = oracle.walk(off, tgt, w, lab, starts, threads=2, **kw)
    np.testing.assert_array_equal(ln, want_len)
    np.testing.assert_array_equal(seq, want_seq)
    np.testing.assert_array_equal(st, want_stats)


def test_oracle_validator(golden):
    case = golden.cases["mp_schema5"]
    off, tgt, w, lab = golden.graph("rmat10")
    starts = golden.starts("mp_schema5")
    seq, ln, _ = golden.expected("mp_schema5")
    assert oracle.validate(off, tgt, lab, starts, seq, ln, case["app"]["schema"]) == 0
    bad = seq.copy()
    i = int(np.flatnonzero(ln >= 2)[0])
    nb = set(tgt[off[seq[i, 0]]:off[seq[i, 0] + 1]].tolist())
    bad[i, 1] = next(x for x in range(len(off) - 1) if x not in nb)  # not an edge
    assert oracle.validate(off, tgt, lab, starts, bad, ln, case["app"]["schema"]) >= 1
    bad2 = seq.copy()
    j = int(np.flatnonzero(ln < 80)[0])
    bad2[j, -1] = 7
    assert oracle.validate(off, tgt, lab, starts, bad2, ln, case["app"]["schema"]) == 1


def test_oracle_thread_count_invariance(golden):
    off, tgt, w, lab = golden.graph("rmat12")
    starts = golden.starts("n2v_rmat12")
    a = oracle.walk(off, tgt, w, lab, starts, app="node2vec", length=24, threads=1)
    b = oracle.walk(off, tgt, w, lab, starts, app="node2vec", length=24, threads=7)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_oracle_matches_reference_on_fuzz_cases():
    """The oracle against the reference's own runs of 200 seeded random
    configurations (tests/golden/fuzz.json): exotic lane widths and
    thresholds, zero weights, self-loops, duplicates, every app."""
    import json

    import fuzz_cases
    import oracle.ingest as ingest
    with open(os.path.join(os.path.dirname(__file__), "golden", "fuzz.json")) as fh:
        ref = {c["seed"]: c for c in json.load(fh)["cases"]}
    for seed in range(fuzz_cases.N_CASES):
        c = fuzz_cases.case(seed)
        off, tgt, w, lab = ingest.build_csr(c["src"], c["dst"], c["w"], c["lab"], c["V"])
        seq, ln, st = oracle.walk(off, tgt, w, lab, c["starts"], k_small=c["eng"]["k_small"],
                                  k_big=c["eng"]["k_big"],
                                  degree_threshold=c["eng"]["degree_threshold"],
                                  sampler=c["eng"]["sampler"], seed=c["seed"], **c["app"])
        want = ref[seed]
        assert fuzz_cases.digest(ln.astype("<u4")) == want["len_sha256"], seed
        assert fuzz_cases.digest(seq.astype("<u4")) == want["seq_sha256"], seed
        assert st.tolist() == want["stats"], seed
