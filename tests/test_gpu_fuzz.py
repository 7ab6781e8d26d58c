"""Seeded random configurations (tests/fuzz_cases.py) on the GPU in all three
summation modes: paths, lengths and the six RunStats counters must equal the
reference's own run of the same case (tests/golden/fuzz.json, written by
tests/golden/gen_fuzz.py from reswalk) and the oracle's."""

import json
import os

import numpy as np
import pytest

import fuzz_cases
import oracle
import paper_2404_08364_b200 as fw

pytestmark = pytest.mark.gpu

STAT_NAMES = ("steps", "edges_scanned", "collectives", "draws", "small_tasks", "large_tasks")
GOLD = os.path.join(os.path.dirname(__file__), "golden", "fuzz.json")


@pytest.fixture(scope="module")
def ref():
    with open(GOLD) as fh:
        return {c["seed"]: c for c in json.load(fh)["cases"]}


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
@pytest.mark.parametrize("seed", range(fuzz_cases.N_CASES))
def test_random_configuration_matches_reference(ref, seed, mode):
    c = fuzz_cases.case(seed)
    g = fw.build_csr(fw.EdgeList(c["src"], c["dst"], c["w"], c["lab"]), c["V"])
    order = "sequential" if mode == "sequential" else "auto"
    env = {"FW_FORCE_CERT": "1"} if mode == "certified" else {}
    seq, ln, st = _run(g, c["starts"], c["app"], c["eng"], c["seed"], order, env)
    want = ref[seed]
    assert fuzz_cases.digest(ln.astype("<u4")) == want["len_sha256"]
    assert fuzz_cases.digest(seq.astype("<u4")) == want["seq_sha256"]
    assert [getattr(st, f) for f in STAT_NAMES] == want["stats"]
    if mode == "auto":  # and the oracle, element by element (readable failures)
        oseq, oln, _ = oracle.walk(g.offsets, g.targets, g.weights, g.labels, c["starts"],
                                   k_small=c["eng"]["k_small"], k_big=c["eng"]["k_big"],
                                   degree_threshold=c["eng"]["degree_threshold"],
                                   sampler=c["eng"]["sampler"], seed=c["seed"], **c["app"])
        np.testing.assert_array_equal(seq, oseq)
