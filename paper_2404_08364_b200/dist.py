"""Multi-GPU data parallelism for the walk path.

In replay mode a query's path is a pure function of (graph, seed, global
qid), so the walk shards into independent queries: every GPU holds a full CSR
replica and walks a disjoint qid range.  No collective is on the walk path.
There are two off-path exchanges:

  * replicate_csr: one source rank's CSR arrays are broadcast to all ranks
    (NCCL over NVLink for cuda tensors; gloo for CPU tensors in tests);
  * gather_paths: the per-rank (sequences, lengths) segments are
    concatenated on the destination rank in qid order.

One process per GPU (torchrun); torch.distributed is plumbing only.
"""

import torch
import torch.distributed as dist


def partition(n, world, rank):
    """Contiguous qid range [lo, hi) of rank `rank` (vertex ids are randomly
    permuted, so contiguous ranges balance in expectation)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def replicate_csr(arrays, shapes_dtypes, src=0, device=None):
    """Broadcast CSR arrays from `src`; other ranks pass arrays=None and get
    freshly allocated tensors of `shapes_dtypes` [(numel, dtype), ...]."""
    rank = dist.get_rank()
    if rank != src:
        # 4 spare elements: the walk kernel reads 16-byte tiles of targets/weights
        arrays = [None if sd is None else
                  torch.empty(sd[0] + 4, dtype=sd[1], device=device)[:sd[0]]
                  for sd in shapes_dtypes]
    for t in arrays:
        if t is not None:
            dist.broadcast(t, src=src)
    return arrays


def gather_paths(seq, lens, n_total, L, dst=0):
    """Concatenate per-rank (seq (n_r*L,), lens (n_r,)) segments on `dst` in
    qid order; returns (seq (n_total, L), lens (n_total,)) on dst, else None.
    Uses all_gather over equal-size padded segments (works on NCCL and gloo)."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    cap = max(partition(n_total, world, r)[1] - partition(n_total, world, r)[0]
              for r in range(world))
    pad_seq = torch.full((cap * L,), -1, dtype=seq.dtype, device=seq.device)
    pad_len = torch.zeros(cap, dtype=lens.dtype, device=lens.device)
    pad_seq[:seq.numel()] = seq
    pad_len[:lens.numel()] = lens
    out_s = [torch.empty_like(pad_seq) for _ in range(world)]
    out_l = [torch.empty_like(pad_len) for _ in range(world)]
    dist.all_gather(out_s, pad_seq)
    dist.all_gather(out_l, pad_len)
    if rank != dst:
        return None
    segs_s, segs_l = [], []
    for r in range(world):
        lo, hi = partition(n_total, world, r)
        segs_s.append(out_s[r][:(hi - lo) * L])
        segs_l.append(out_l[r][:hi - lo])
    return torch.cat(segs_s).view(n_total, L), torch.cat(segs_l)
