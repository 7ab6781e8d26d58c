"""CPU-side tests: C-ABI library loads and exports every declared symbol,
host API validation (same exceptions as the reference), graph I/O, the
synthetic R-MAT generator, and no silent CPU fallback."""

import os
import re

import numpy as np
import pytest

import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import _lib, rmat
from paper_2404_08364_b200.engine import batch_size

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_library_exports_every_declared_symbol():
    with open(os.path.join(ROOT, "include", "flowwalk.h")) as fh:
        header = fh.read()
    declared = set(re.findall(r"^\s*(?:int|const char \*)\s*(fw_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTS)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name


def test_engine_config_validation():
    for bad in (dict(workers=0), dict(local_pool=0), dict(k_small=64, k_big=32),
                dict(sampler="bogus"), dict(k_big=1001), dict(degree_threshold=0),
                dict(order="fast"), dict(devices=())):
        with pytest.raises(fw.ConfigError):
            fw.EngineConfig(**bad).validate()
    cfg = fw.EngineConfig()
    assert cfg.resolve_sampler("node2vec") == 1
    assert cfg.resolve_sampler("deepwalk") == 0
    assert fw.EngineConfig(sampler="dprs").resolve_sampler("ppr") == 1


def test_app_config_validation():
    for bad in (dict(app="x"), dict(length=0), dict(app="ppr", stop_prob=1.5),
                dict(app="node2vec", a=0), dict(app="metapath", schema=())):
        with pytest.raises(fw.ValidationError):
            fw.AppConfig(**bad).validate()


def test_batch_size_eq3():
    assert batch_size(fw.EngineConfig(memory_budget=800, graph_bytes=0), 99) == 1
    assert batch_size(fw.EngineConfig(memory_budget=8_000_000, graph_bytes=0), 79) == 12_500
    with pytest.raises(fw.ConfigError):
        batch_size(fw.EngineConfig(memory_budget=100, graph_bytes=100), 10)
    with pytest.raises(fw.ConfigError):
        batch_size(fw.EngineConfig(), 10)


def test_validation_happens_before_device(golden):
    off, tgt, w, lab = golden.graph("rmat10")
    g = fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)
    with pytest.raises(fw.ValidationError):
        list(fw.run_batches(g, np.array([g.vertex_count]), fw.AppConfig(), fw.EngineConfig()))
    with pytest.raises(fw.ConfigError):
        list(fw.run_batches(g, np.array([0]), fw.AppConfig(length=1 << 20), fw.EngineConfig()))


@pytest.mark.skipif(_lib.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(golden):
    off, tgt, w, lab = golden.graph("rmat10")
    g = fw.Graph(len(off) - 1, len(tgt), off, tgt, w, lab)
    with pytest.raises(_lib.FlowWalkUnavailable):
        fw.run(g, np.arange(10), fw.AppConfig(), fw.EngineConfig(replay=True))


def test_graph_binary_roundtrip(tmp_path):
    g = rmat.rmat_graph(8)
    p = tmp_path / "g.fwg"
    fw.save_binary(g, p)
    h = fw.load_binary(p)
    for a in ("offsets", "targets", "weights", "labels"):
        np.testing.assert_array_equal(getattr(g, a), getattr(h, a))
    blob = bytearray(p.read_bytes())
    blob[40] ^= 1
    p.write_bytes(bytes(blob))
    with pytest.raises(fw.FormatError):
        fw.load_binary(p)


def test_parse_and_build_csr():
    g = fw.build_csr(fw.parse_edge_list("0 2 3.0 1\n0 1\n1 0\n# c\n0 1 2.0"), 3)
    assert g.offsets.tolist() == [0, 3, 4, 4]
    assert g.targets.tolist() == [1, 1, 2, 0]
    assert g.weights.tolist() == [1.0, 2.0, 3.0, 1.0]  # stable among duplicates
    with pytest.raises(fw.ParseError):
        fw.parse_edge_list("0 1 2 3 4")
    with pytest.raises(fw.ValidationError):
        fw.parse_edge_list("0 1 -1")


def test_rmat_host_properties():
    g = rmat.rmat_graph(12)
    assert g.vertex_count == 4096 and g.edge_count == 16 * 4096
    g.validate()
    # symmetric: the multiset of (u, v) equals that of (v, u)
    src = np.repeat(np.arange(g.vertex_count), np.diff(g.offsets))
    a = np.sort(src.astype(np.int64) << 32 | g.targets)
    b = np.sort(g.targets.astype(np.int64) << 32 | src)
    np.testing.assert_array_equal(a, b)
    for v in range(0, g.vertex_count, 97):  # neighbour lists sorted
        nb = g.neighbors(v)
        assert np.all(nb[1:] >= nb[:-1])
    assert g.weights.min() >= 1.0 and g.weights.max() < 5.0
    assert set(np.unique(g.labels).tolist()) == {0, 1, 2, 3, 4}
    # power law: heavy hub, many isolated vertices
    deg = np.diff(g.offsets)
    assert deg.max() > 50 * deg.mean() and (deg == 0).mean() > 0.2
    h = rmat.rmat_graph(12)
    np.testing.assert_array_equal(g.targets, h.targets)


def test_perm_bits_is_bijective():
    for s in (1, 5, 10, 16):
        x = np.arange(1 << s, dtype=np.uint64)
        assert len(np.unique(rmat.perm_bits(x, s, 12345))) == 1 << s


def test_alias_table_matches_reference(golden):
    """trials.alias_table restates samplers.alias_build (samplers.py:245-266)."""
    from paper_2404_08364_b200.trials import alias_table
    for v in {c["vec"] for c in golden.trials}:
        prob, alias = alias_table(golden.z[f"t_w_{v}"])
        np.testing.assert_array_equal(prob, golden.z[f"t_aliasprob_{v}"])
        np.testing.assert_array_equal(alias, golden.z[f"t_aliasidx_{v}"])
