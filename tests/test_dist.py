"""World-size-2 gloo test of the multi-GPU host logic (CSR replication,
qid partitioning, path gather).  The per-rank walker here is the CPU oracle
standing in for the device kernel, so the test runs without a GPU; the GPU
path shares the same partition/offset code (bench.py, engine.py)."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2404_08364_b200 import dist as fwd
    from paper_2404_08364_b200 import rmat
    L = 16
    if rank == 0:
        g = rmat.rmat_graph(11)
        arrays = [torch.from_numpy(g.offsets), torch.from_numpy(g.targets.view(np.int32)),
                  torch.from_numpy(g.weights)]
        V, E = g.vertex_count, g.edge_count
        meta = torch.tensor([V, E], dtype=torch.int64)
    else:
        arrays, meta = None, torch.zeros(2, dtype=torch.int64)
    dist.broadcast(meta, src=0)
    V, E = (int(x) for x in meta)
    arrays = fwd.replicate_csr(arrays, [(V + 1, torch.int64), (E, torch.int32),
                                        (E, torch.float32)], src=0)
    off, tgt, w = (a.numpy() for a in arrays)
    n = V
    lo, hi = fwd.partition(n, world, rank)
    starts = np.arange(lo, hi, dtype=np.int64)
    seq, ln, _ = oracle.walk(off, tgt.view(np.uint32), w, None, starts, app="node2vec",
                             length=L, base_qid=lo, threads=1)
    res = fwd.gather_paths(torch.from_numpy(seq.reshape(-1).view(np.int32)),
                           torch.from_numpy(ln.view(np.int32)), n, L, dst=0)
    if rank == 0:
        full_seq, full_len, _ = oracle.walk(off, tgt.view(np.uint32), w, None,
                                            np.arange(n, dtype=np.int64), app="node2vec",
                                            length=L, threads=2)
        ok = (np.array_equal(res[0].numpy().view(np.uint32), full_seq)
              and np.array_equal(res[1].numpy().view(np.uint32), full_len))
        with open(out_path, "w") as fh:
            fh.write("ok" if ok else "mismatch")
    dist.barrier()
    dist.destroy_process_group()


def test_partition_covers_range():
    from paper_2404_08364_b200.dist import partition
    for n in (0, 1, 7, 1000, 4194304):
        for world in (1, 2, 3, 8):
            parts = [partition(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))


def test_two_rank_replicate_partition_gather(tmp_path):
    out = tmp_path / "res.txt"
    mp.spawn(_worker, args=(2, _free_port(), str(out)), nprocs=2, join=True)
    assert out.read_text() == "ok"
