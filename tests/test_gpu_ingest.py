"""Graph ingest on the GPU: build_csr by the device radix
sort and load_binary by the streamed FWG1 reader with a device CRC-32, pinned
against reswalk's own outputs (tests/golden/ingest.npz, ref_graph.fwg) and the
oracle's lexsort restatement (oracle/ingest.py) on larger inputs."""

import ctypes
import os
import zlib

import numpy as np
import pytest

import oracle
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import _lib, rmat

pytestmark = pytest.mark.gpu

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
GOLD = os.path.join(ROOT, "tests", "golden")
INGEST_CASES = ["dups64", "zipf17", "star", "empty", "parsed_undirected"]


@pytest.fixture(scope="module")
def z():
    return np.load(os.path.join(GOLD, "ingest.npz"))


def _edges(z, name):
    return fw.EdgeList(z[f"in_{name}_src"], z[f"in_{name}_dst"], z[f"in_{name}_w"],
                       z[f"in_{name}_lab"])


def _assert_graph(g, offsets, targets, weights, labels):
    np.testing.assert_array_equal(g.offsets, offsets)
    np.testing.assert_array_equal(g.targets, targets)
    np.testing.assert_array_equal(g.weights, weights)
    np.testing.assert_array_equal(g.labels, labels)


@pytest.mark.parametrize("name", INGEST_CASES)
def test_build_csr_equals_reference(z, name):
    vc = int(z[f"in_{name}_vc"])
    g = fw.build_csr(_edges(z, name), None if vc < 0 else vc)
    _assert_graph(g, *(z[f"out_{name}_{k}"] for k in ("offsets", "targets", "weights", "labels")))
    assert g.vertex_count == len(z[f"out_{name}_offsets"]) - 1


@pytest.mark.parametrize("V,m,seed", [(1 << 20, 1 << 23, 1), (3 << 24, 1 << 22, 2),
                                      (1, 1000, 3), (2, 77777, 4), ((1 << 31) + 12345, 5000, 5)])
def test_build_csr_device_equals_lexsort(V, m, seed):
    """Larger inputs against the oracle's np.lexsort restatement: many
    duplicates (V = 1, 2), 52-bit keys (V = 3 * 2^24), 64-bit keys with the
    top ids (V = 2^31 + 12345, ids drawn near both ends)."""
    rs = np.random.default_rng(seed)
    if V > 1 << 31:
        pool = np.concatenate([np.arange(50), V - 1 - np.arange(50)]).astype(np.uint32)
        src, dst = rs.choice(pool, m), rs.choice(pool, m)
    else:
        src = rs.integers(0, V, m).astype(np.uint32)
        dst = rs.integers(0, V, m).astype(np.uint32)
    w = rs.random(m).astype(np.float32)
    lab = rs.integers(0, 256, m).astype(np.uint8)
    el = fw.EdgeList(src, dst, w, lab)
    if V > 1 << 28:  # too many offsets for a host copy: check the sorted arrays only
        dg = fw.build_csr_device(el, V)
        want = oracle.ingest.build_csr(src, dst, w, lab, int(max(src.max(), dst.max())) + 1)
        np.testing.assert_array_equal(dg.targets.cpu().numpy().view(np.uint32), want[1])
        np.testing.assert_array_equal(dg.weights.cpu().numpy(), want[2])
        np.testing.assert_array_equal(dg.labels.cpu().numpy(), want[3])
        off = dg.offsets
        np.testing.assert_array_equal(off[pool_ids(src, dst)].cpu().numpy(),
                                      _offsets_at(src, pool_ids(src, dst)))
        assert int(off[-1].item()) == m
        dg.close()
        return
    g = fw.build_csr(el, V)
    _assert_graph(g, *oracle.ingest.build_csr(src, dst, w, lab, V))


def pool_ids(src, dst):
    import torch
    ids = np.unique(np.concatenate([src, dst]).astype(np.int64))
    return torch.from_numpy(np.concatenate([ids, ids + 1])).cuda()


def _offsets_at(src, ids_t):
    ids = ids_t.cpu().numpy()
    s = np.sort(src.astype(np.int64))
    return np.searchsorted(s, ids, side="left")


def test_build_csr_errors_and_inference(z):
    el = fw.EdgeList(np.array([0, 9], np.uint32), np.array([3, 1], np.uint32),
                     np.ones(2, np.float32), np.zeros(2, np.uint8))
    with pytest.raises(fw.ValidationError, match="out of range"):
        fw.build_csr(el, 5)
    with pytest.raises(fw.ValidationError, match="out of range"):
        fw.build_csr_device(el, 9)
    g = fw.build_csr(el)
    assert g.vertex_count == 10 and g.offsets.tolist() == [0, 1] + [1] * 8 + [2]
    bad = fw.EdgeList(el.src, el.dst, np.array([1.0, -1.0], np.float32), el.label)
    with pytest.raises(fw.ValidationError, match="weights"):
        fw.build_csr(bad)


@pytest.mark.parametrize("scale", [10, 17])
def test_build_csr_device_walks_like_host_build(scale):
    """A graph built on the device walks exactly like the same graph built by
    the oracle's lexsort (Node2Vec needs the sorted lists)."""
    u, v = rmat.rmat_edges_host(scale, 8 << scale, seed=9)
    src, dst = np.concatenate([u, v]), np.concatenate([v, u])
    w = rmat.synth_weights_host(4, 0, len(src))
    el = fw.EdgeList(src, dst, w, np.zeros(len(src), np.uint8))
    dg = fw.build_csr_device(el, 1 << scale)
    off, tgt, ww, _ = oracle.ingest.build_csr(src, dst, w, el.label, 1 << scale)
    starts = np.arange(min(1 << scale, 20000), dtype=np.int64)
    seqs = []
    fw.run(dg, starts, fw.AppConfig(app="node2vec", length=20), fw.EngineConfig(replay=True),
           sink=lambda b: seqs.append(b.sequences.copy()))
    oseq, _oln, _ = oracle.walk(off, tgt, ww, None, starts, app="node2vec", length=20)
    np.testing.assert_array_equal(np.concatenate(seqs), oseq)
    dg.close()


def test_load_binary_reads_reference_file(z):
    """A file written by reswalk.save_binary loads (device CRC check passes)
    into the reference's arrays."""
    g = fw.load_binary(os.path.join(GOLD, "ref_graph.fwg"))
    _assert_graph(g, *(z[f"out_dups64_{k}"] for k in ("offsets", "targets", "weights", "labels")))


def test_load_binary_device_large_and_corrupt(tmp_path):
    """R-MAT s20 (~150 MB: many 32 MB chunks over the reader threads) round
    trip, then the reference's FormatError cases: bad magic, truncation,
    one flipped payload byte (checksum)."""
    g = rmat.rmat_graph(20)
    p = tmp_path / "s20.fwg"
    fw.save_binary(g, p)
    dg = fw.load_binary_device(p)
    h = dg.to_host()
    _assert_graph(h, g.offsets, g.targets, g.weights, g.labels)
    assert dg.max_degree() == g.max_degree()
    dg.close()
    blob = bytearray(p.read_bytes())
    for name, data, msg in (
            ("magic", b"FWG2" + bytes(blob[4:]), "bad magic"),
            ("short", bytes(blob[:-1]), "truncated"),
            ("flip", bytes(blob[:1000]) + bytes([blob[1000] ^ 0x10]) + bytes(blob[1001:]),
             "checksum"),
            ("flip_tail", bytes(blob[:-7]) + bytes([blob[-7] ^ 1]) + bytes(blob[-6:]),
             "checksum")):
        q = tmp_path / f"{name}.fwg"
        q.write_bytes(data)
        with pytest.raises(fw.FormatError, match=msg):
            fw.load_binary_device(q)


def test_load_binary_rejects_invalid_csr(tmp_path):
    """A well-formed file whose CSR is invalid raises ValidationError after
    the format checks (load_binary ends with Graph.validate)."""
    off = np.array([0, 2, 3], np.int64)
    for tgt, w, msg in ((np.array([1, 7, 0], np.uint32), np.ones(3, np.float32), "target"),
                        (np.array([1, 1, 0], np.uint32), np.array([1, -2, 1], np.float32),
                         "weights")):
        g = fw.Graph(2, 3, off, tgt, w)
        p = tmp_path / "bad.fwg"
        fw.save_binary(g, p)
        with pytest.raises(fw.ValidationError, match=msg):
            fw.load_binary(p)


@pytest.mark.parametrize("n,shift", [(0, 0), (1, 0), (4095, 0), (4096, 0), (4097, 0),
                                     (1_000_003, 0), (65536 * 3 + 5, 3), (12_345_678, 16)])
def test_device_crc32_equals_zlib(n, shift):
    import torch
    rs = np.random.default_rng(n)
    host = rs.integers(0, 256, n + shift, dtype=np.uint8)
    d = torch.from_numpy(host).cuda()
    out = ctypes.c_uint32()
    _lib.check(_lib.load().fw_crc32_device(d.data_ptr() + shift if n else None, n,
                                           ctypes.byref(out), None))
    assert out.value == zlib.crc32(host[shift:].tobytes()) & 0xFFFFFFFF


@pytest.mark.parametrize("with_w", [True, False])
def test_build_csr_device_without_labels(with_w):
    """The sort's value variants: weights without labels ride through the sort
    as the value (no gather), and with neither only the keys move (weights 1)."""
    import torch
    rs = np.random.default_rng(11)
    V, m = 1 << 16, 1 << 21
    src = rs.integers(0, V, m).astype(np.uint32)
    dst = rs.integers(0, V, m).astype(np.uint32)
    w = rs.random(m).astype(np.float32)
    d = torch.device("cuda", 0)
    t = (torch.from_numpy(src.view(np.int32)).to(d), torch.from_numpy(dst.view(np.int32)).to(d),
         torch.from_numpy(w).to(d) if with_w else None, None)
    dg = fw.build_csr_device(t, V)
    want = oracle.ingest.build_csr(src, dst, w if with_w else np.ones(m, np.float32),
                                   np.zeros(m, np.uint8), V)
    np.testing.assert_array_equal(dg.offsets.cpu().numpy(), want[0])
    np.testing.assert_array_equal(dg.targets.cpu().numpy().view(np.uint32), want[1])
    np.testing.assert_array_equal(dg.weights.cpu().numpy(), want[2])
    assert dg.labels is None
    dg.close()
