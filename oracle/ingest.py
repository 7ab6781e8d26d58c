"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference's graph ingest.

``build_csr`` follows reswalk ``graph.build_csr`` (graph.py:138-169): vertex
count inferred as max id + 1 when omitted, neighbour lists ordered by
``np.lexsort((dst, src))`` (stable: duplicate (src, dst) pairs keep their
input order), offsets from a bincount of the sources.  ``crc32`` is zlib's,
which the reference's FWG1 writer/reader use (graph.py:213-216, 241-244).
Pinned against tests/golden/ingest.npz, produced by running reswalk itself
(tests/golden/gen_ingest.py).
"""

import zlib

import numpy as np


def build_csr(src, dst, weight, label, vertex_count=None):
    src = np.asarray(src, np.uint32)
    dst = np.asarray(dst, np.uint32)
    m = len(src)
    if vertex_count is None:
        vertex_count = int(max(src.max(), dst.max())) + 1 if m else 0
    order = np.lexsort((dst, src))
    offsets = np.zeros(vertex_count + 1, np.int64)
    if m:
        offsets[1:] = np.cumsum(np.bincount(src, minlength=vertex_count))
    return (offsets, dst[order].astype(np.uint32), np.asarray(weight, np.float32)[order],
            np.asarray(label, np.uint8)[order])


def crc32(buf):
    return zlib.crc32(buf) & 0xFFFFFFFF
