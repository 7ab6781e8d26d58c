"""Synthetic Graph500 R-MAT workload (BASELINE.json configs).

The reference ships no R-MAT generator (only uniform/star edge lists,
graph.py:257-277), so the workload is defined here: edge-factor-16
symmetrised R-MAT with (a, b, c, d) = (0.57, 0.19, 0.19, 0.05), vertex ids
scrambled by a bijective hash, duplicates and self-loops kept, neighbour
lists sorted; weights U[1,5) float32 and labels U{0..4} uint8 assigned per
CSR position.  Every random choice is a counter hash (the walk RNG's mix64),
so the numpy path here and the device path (fw_rmat_edges_device &c. in
csrc/fw_api.cu) produce identical arrays; tests pin that on small scales.
The oracle always receives the exact arrays the GPU walks.  The device
build sorts with the library's own radix sort (fw_build_csr_device).
"""

import numpy as np

from .graph import Graph
from .rng import GOLDEN, MASK64, MIX1, MIX2, mix64, mix64_np

RMAT_ABC = (0.57, 0.19, 0.19)
GRAPH_SEED, WEIGHT_SEED, LABEL_SEED = 1, 2, 3


def _thresh(p):
    if p <= 0:
        return 0
    t = int(np.floor(p * 4294967296.0))
    return min(t, 0xFFFFFFFF)


def perm_bits(x, s, key):
    """Bijection on [0, 2^s): xor key, then (odd multiply, xorshift) x 3."""
    x = np.asarray(x, dtype=np.uint64)
    if s == 0:
        return np.zeros_like(x)
    mask = np.uint64((1 << s) - 1)
    sh = np.uint64((s + 1) // 2)
    with np.errstate(over="ignore"):
        x = (x ^ np.uint64(key)) & mask
        for mul in (GOLDEN, MIX1, MIX2):
            x = (x * np.uint64(mul)) & mask
            x ^= x >> sh
    return x


def rmat_edges_host(scale, m, seed=GRAPH_SEED, abc=RMAT_ABC, e0=0):
    """(src, dst) uint32 of R-MAT edges e0 .. e0+m-1 (numpy twin of k_rmat)."""
    a, b, c = abc
    ta, tab, tabc = _thresh(a), _thresh(a + b), _thresh(a + b + c)
    h = np.uint64(mix64(seed + GOLDEN))
    pkey = mix64(seed ^ 0x5555555555555555)
    e = np.arange(e0, e0 + m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = mix64_np(h ^ (e * np.uint64(MIX1)))
        u = np.zeros(m, np.uint64)
        v = np.zeros(m, np.uint64)
        for lvl in range(scale):
            r = (mix64_np(base + np.uint64((lvl * GOLDEN) & MASK64)) >> np.uint64(32))
            sb = r >= tab
            db = ((r >= ta) & (r < tab)) | (r >= tabc)
            u = (u << np.uint64(1)) | sb.astype(np.uint64)
            v = (v << np.uint64(1)) | db.astype(np.uint64)
    return (perm_bits(u, scale, pkey).astype(np.uint32),
            perm_bits(v, scale, pkey).astype(np.uint32))


def synth_weights_host(seed, e0, m):
    h = np.uint64(mix64(seed + GOLDEN))
    e = np.arange(e0, e0 + m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = mix64_np(h + e * np.uint64(GOLDEN))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / (1 << 53))
    w = (1.0 + 4.0 * u).astype(np.float32)
    w[w >= np.float32(5.0)] = np.nextafter(np.float32(5.0), np.float32(1.0))
    return w


def synth_labels_host(seed, label_count, e0, m):
    h = np.uint64(mix64(seed + GOLDEN))
    e = np.arange(e0, e0 + m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = mix64_np(h + e * np.uint64(GOLDEN))
    return ((z >> np.uint64(32)) % np.uint64(label_count)).astype(np.uint8)


def rmat_graph(scale, edge_factor=16, seed=GRAPH_SEED, labels=True,
               weight_seed=WEIGHT_SEED, label_seed=LABEL_SEED, label_count=5):
    """Host (numpy) build; fine up to scale ~20.  E = edge_factor * 2^scale."""
    V = 1 << scale
    m = edge_factor * V // 2
    u, v = rmat_edges_host(scale, m, seed)
    key = np.concatenate([u, v]).astype(np.uint64) << np.uint64(32)
    key |= np.concatenate([v, u]).astype(np.uint64)
    key.sort()
    src = (key >> np.uint64(32)).astype(np.int64)
    targets = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    E = len(targets)
    offsets = np.zeros(V + 1, np.int64)
    np.cumsum(np.bincount(src, minlength=V), out=offsets[1:])
    w = synth_weights_host(weight_seed, 0, E)
    lab = synth_labels_host(label_seed, label_count, 0, E) if labels else None
    return Graph(V, E, offsets, targets, w, lab)


def rmat_graph_device(scale, edge_factor=16, seed=GRAPH_SEED, labels=True,
                      weight_seed=WEIGHT_SEED, label_seed=LABEL_SEED, label_count=5,
                      device=0):
    """Device build: hash-generated edges and both directions of each
    (fw_rmat_edges_device, called twice with the outputs swapped), CSR by the
    device build_csr (fw_build_csr_device: stable radix sort), weights and
    labels by CSR position.  Returns a DeviceGraph whose arrays equal
    rmat_graph(...)'s."""
    import torch

    from . import _lib
    from .engine import DeviceGraph

    lib = _lib.load()
    dev = torch.device("cuda", device)
    V = 1 << scale
    m = edge_factor * V // 2
    E = 2 * m
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev).cuda_stream
        src = torch.empty(E, dtype=torch.int32, device=dev)
        dst = torch.empty(E, dtype=torch.int32, device=dev)
        _lib.check(lib.fw_rmat_edges_device(seed, scale, *RMAT_ABC, 0, m, src.data_ptr(),
                                            dst.data_ptr(), stream))
        _lib.check(lib.fw_rmat_edges_device(seed, scale, *RMAT_ABC, 0, m, dst.data_ptr() + 4 * m,
                                            src.data_ptr() + 4 * m, stream))
        offsets = torch.empty(V + 1, dtype=torch.int64, device=dev)
        # +4 elements: the walk kernel reads 16-byte tiles (DeviceGraph contract)
        targets = torch.empty(E + 4, dtype=torch.int32, device=dev)[:E]
        _lib.check(lib.fw_build_csr_device(src.data_ptr(), dst.data_ptr(), None, None, E, V,
                                           offsets.data_ptr(), targets.data_ptr(), None, None,
                                           stream))
        del src, dst
        weights = torch.empty(E + 4, dtype=torch.float32, device=dev)[:E]
        _lib.check(lib.fw_synth_weights_device(weight_seed, 0, E, weights.data_ptr(), stream))
        lab = None
        if labels:
            lab = torch.empty(E, dtype=torch.uint8, device=dev)
            _lib.check(lib.fw_synth_labels_device(label_seed, label_count, 0, E,
                                                  lab.data_ptr(), stream))
        torch.cuda.synchronize(dev)
    return DeviceGraph(V, E, offsets, targets, weights, lab, device=device)
