"""Multi-GPU data parallelism for the walk path.

In replay mode a query's path is a pure function of (graph, seed, global
qid), so the walk shards into independent queries: every GPU holds a full CSR
replica and walks a disjoint qid range.  No collective is on the walk path.
There are two off-path exchanges:

  * replicate_csr: one source rank's CSR arrays are broadcast to all ranks
    (NCCL over NVLink for cuda tensors; gloo for CPU tensors in tests);
  * gather_paths: the per-rank (sequences, lengths) segments are sent
    point-to-point to the destination rank, in qid order;
  * share_buffers (the default in bench.py): no gather phase at all -- the
    destination rank exports its result buffers by CUDA IPC and every rank's
    walk kernel stores its path rows straight into them (NVLink peer stores,
    fused with the walk; the rows are ~1 GB/s per GPU against 900 GB/s links).

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
    """Point-to-point gather of the per-rank path segments to `dst`, in qid
    order: every other rank sends its (seq (n_r*L,), lens (n_r,)) segment
    straight into its slice of dst's output (NCCL send/recv over NVLink for
    cuda tensors, gloo for CPU tensors).  Only dst holds the full result
    (an all-gather would land n_total*L*4 bytes on every rank).  Returns
    (seq (n_total, L), lens (n_total,)) on dst, else None."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    if rank != dst:
        if seq.numel():
            reqs = [dist.isend(seq.contiguous(), dst), dist.isend(lens.contiguous(), dst)]
            for r in reqs:
                r.wait()
        return None
    out_s = torch.empty(n_total * L, dtype=seq.dtype, device=seq.device)
    out_l = torch.empty(n_total, dtype=lens.dtype, device=lens.device)
    lo, hi = partition(n_total, world, rank)
    out_s[lo * L:hi * L] = seq
    out_l[lo:hi] = lens
    reqs = []
    for r in range(world):
        lo, hi = partition(n_total, world, r)
        if r == rank or hi == lo:
            continue
        reqs.append(dist.irecv(out_s[lo * L:hi * L], r))
        reqs.append(dist.irecv(out_l[lo:hi], r))
    for q in reqs:
        q.wait()
    return out_s.view(n_total, L), out_l


def share_buffers(tensors, src=0):
    """CUDA IPC: rank `src` exports its device tensors and every other rank
    gets views of the same memory (opened with lazy peer access, so a kernel
    on another GPU stores into it over NVLink; on one GPU it is plain shared
    device memory).  Returns the list of tensors (src: its own).  The views
    must be dropped before `src` frees the originals (call
    release_shared() then barrier)."""
    rank = dist.get_rank()
    obj = [None]
    if rank == src:
        obj = [[(t.untyped_storage()._share_cuda_(), t.dtype, t.numel(), t.storage_offset())
                for t in tensors]]
    dist.broadcast_object_list(obj, src=src)
    if rank == src:
        return list(tensors)
    views = []
    for handle, dtype, numel, offset in obj[0]:
        st = torch.UntypedStorage._new_shared_cuda(*handle)
        dev = torch.device("cuda", handle[0])
        views.append(torch.empty(0, dtype=dtype, device=dev).set_(st, offset, (numel,), (1,)))
    return views
