#!/usr/bin/env python
"""Walk-engine benchmark (driver contract; BASELINE.json metric).

Default workload = BASELINE.json configs[1]: Node2Vec (a=2, b=0.5, L=80),
one query per vertex, synthetic R-MAT scale-22 edge-factor-16 graph, replay
mode, seed 0.  A "step" is one pass of the walk kernel over all V queries.

  value        sampled steps/s (sum of walk lengths / device time), inputs
               resident in HBM, CUDA events on the launching stream, max over
               ranks; graph + result pool (1.9 GB) exceed L2, so no flush.
  e2e          the same metric through the C-ABI host-buffer call fw_walk
               (H2D of the starts from pinned memory, D2H of sequences+lengths
               into pinned memory inside the timed region; fw_walk copies the
               result back in 16 pieces, each as soon as its queries finish).
  roofline     algorithmic bytes per launch / mean launch time vs
               the measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline the reference itself (baseline/_ref reswalk, numba, all host
               threads) on a bounded sample of the same workload (rank 0, N=1).

--impl reference times the reference's CPU implementation the same way
(rank 0 only; other ranks exit 0).  Multi-GPU (torchrun): the
graph is generated on rank 0 and broadcast over NCCL (off the timed path);
ONE query set (one query per vertex) is partitioned into contiguous global-qid
ranges, one per rank (strong scaling; --scaling weak gives every rank its own
full query set instead).  No collective runs on the walk path; `value` is all
ranks' sampled steps over the max-over-ranks device time.  After the timed
region the path segments are gathered point-to-point to rank 0 (NCCL
send/recv over NVLink), timed separately (config.gather_ms).
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REASON_FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--scale", type=int, default=22)
    p.add_argument("--app", default="node2vec",
                   choices=["node2vec", "deepwalk", "ppr", "metapath"])
    p.add_argument("--length", type=int, default=None)
    p.add_argument("--queries", default="all", help="all | hub (PPR config)")
    p.add_argument("--a", type=float, default=2.0, help="node2vec return parameter (p)")
    p.add_argument("--b", type=float, default=0.5, help="node2vec in-out parameter (q)")
    p.add_argument("--weights", choices=["uniform", "lognormal"], default="uniform",
                   help="edge weights: U[1,5) (BASELINE) or log-normal(0, 1) as "
                        "graph.py:183-188 draws them (seed 2): sums that round, the "
                        "certified-summation path")
    p.add_argument("--sampler", choices=["auto", "dprs", "zprs"], default="auto",
                   help="EngineConfig.sampler (auto: DPRS for Node2Vec, else ZPRS)")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--nq", type=int, default=0,
                   help="queries (0 = one per vertex; 2^24 for scale >= 26, so one step of "
                        "the s27 workload stays ~17 s on one GPU)")
    p.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                   help="strong: one query set partitioned over the GPUs (default); "
                        "weak: every GPU walks its own full query set (disjoint global qids)")
    p.add_argument("--gather", choices=["direct", "nccl", "none"], default="direct",
                   help="N>1 strong scaling: how the paths reach rank 0. direct: every rank's "
                        "walk kernel stores its rows straight into rank 0's buffer (CUDA IPC, "
                        "NVLink peer stores, no gather phase); nccl: point-to-point NCCL "
                        "send/recv after the walk, timed separately; none")
    p.add_argument("--no-gather", action="store_true", help="same as --gather none")
    p.add_argument("--dump-gather", default=None,
                   help="N>1: rank 0 saves the gathered paths (.npz) for tests")
    return p.parse_args()


def app_config(args):
    import paper_2404_08364_b200 as fw
    if args.app == "node2vec":
        return fw.AppConfig(app="node2vec", length=args.length or 80, a=args.a, b=args.b)
    if args.app == "deepwalk":
        return fw.AppConfig(app="deepwalk", length=args.length or 80)
    if args.app == "ppr":
        return fw.AppConfig(app="ppr", length=args.length or 80, stop_prob=0.2)
    return fw.AppConfig(app="metapath", length=args.length or 5, schema=(0, 1, 2, 3, 4))


def metric_name(args):
    names = {"node2vec": "Node2Vec", "deepwalk": "DeepWalk", "ppr": "PPR", "metapath": "MetaPath"}
    return f"{names[args.app]} sampled steps/sec"


def workload_name(args, app):
    extra = {"node2vec": f" p={args.a:g} q={args.b:g}", "ppr": " stop 0.2", "metapath": " schema 0..4",
             "deepwalk": " weighted"}[args.app]
    q = "all queries at the max-degree vertex" if args.queries == "hub" else "one query per vertex"
    wt = ", log-normal weights" if args.weights == "lognormal" else ""
    return f"{metric_name(args).split()[0]}{extra} length {app.length}, {q}, R-MAT scale-{args.scale} ef16{wt}"


def workload_config(args, app, world):
    """The workload-defining `config` object, identical for both arms (the
    measurement outputs of a run go under "run")."""
    V = 1 << args.scale
    n_total = args.nq if args.nq else (V if args.scale < 26 else 1 << 24)
    if args.scaling == "strong":
        per_gpu = n_total // world  # rank 0's share (dist.partition)
        total = n_total
    else:
        per_gpu, total = n_total, n_total * world
    return {"workload": workload_name(args, app), "graph": f"rmat-s{args.scale}-ef16",
            "sampler": args.sampler, "weights": args.weights, "vertices": V,
            "csr_entries": 16 * V, "queries_per_gpu": per_gpu, "total_queries": total,
            "parallelism": f"replicated graph, qids partitioned x{world}",
            "l2": "inputs larger than L2 (graph + result pool > 126 MB), no flush"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             + ",".join(f"clocks_event_reasons.{r}" for r in REASON_FIELDS))
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 5 + len(REASON_FIELDS):
                    continue
                try:
                    sm.append(float(f[1]))
                    mx.append(float(f[2]))
                except ValueError:
                    continue
                for name, val in zip(REASON_FIELDS, f[5:]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(workload, alg_bytes):
    """DRAM bytes per launch of the walk kernel, from the committed ncu
    --set full capture of this workload (profiles/walk_traffic.json).  The
    capture runs a smaller launch (fewer queries) to keep ncu's replays
    short, so it is scaled by the ratio of algorithmic bytes."""
    try:
        with open(os.path.join(ROOT, "profiles", "walk_traffic.json")) as fh:
            d = json.load(fh).get(workload)
    except (OSError, ValueError):
        return None, None
    if not d or not d.get("alg_bytes"):
        return None, None
    return (d["dram_bytes"] * alg_bytes / d["alg_bytes"],
            f"ncu --set full of a {d['queries']}-query launch ({d['report']}): "
            f"{d['dram_bytes'] / d['alg_bytes']:.3f} DRAM bytes per algorithmic byte, "
            f"scaled to this launch")


def profiled_counters(workload):
    """What bounds the kernel, from the same committed capture: issue-slot
    use, L2 sector throughput and global-load sector efficiency."""
    try:
        with open(os.path.join(ROOT, "profiles", "walk_traffic.json")) as fh:
            d = json.load(fh).get(workload) or {}
    except (OSError, ValueError):
        return None
    if "issue_pct" not in d:
        return None
    return {"issue_slots_busy_pct": d["issue_pct"],
            "l2_sector_throughput_pct_of_peak": d.get("l2_sector_pct_of_peak"),
            "global_load_bytes_used_per_32B_sector": d.get("sector_bytes_used"),
            "dram_bytes_per_algorithmic_byte": d["dram_bytes"] / d["alg_bytes"],
            "report": d["report"]}


# ---------------------------------------------------------------------------
# CPU reference (baseline/_ref reswalk) on a bounded sample
# ---------------------------------------------------------------------------
def import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "nbc_ref"))
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "reswalk")) and ref not in sys.path:
        sys.path.insert(0, ref)
    import reswalk  # noqa: F401
    from reswalk import engine as E
    from reswalk.apps import AppConfig
    from reswalk.graph import Graph
    return E, AppConfig, Graph


def reference_runner(host_graph, app, starts_all, sampler="auto"):
    """Returns (kind, run(n, offset) -> (sampled_steps, seconds), cores)."""
    cores = os.cpu_count() or 1
    try:
        E, RAppConfig, RGraph = import_reference()
        rg = RGraph(host_graph.vertex_count, host_graph.edge_count, host_graph.offsets,
                    host_graph.targets, host_graph.weights, host_graph.labels)
        rapp = RAppConfig(app=app.app, length=app.length, stop_prob=app.stop_prob, a=app.a,
                          b=app.b, schema=tuple(app.schema), weighted=app.weighted)
        eng = E.EngineConfig(workers=cores, replay=True, sampler=sampler)

        def run(n, off):
            total = [0]

            def sink(b):
                total[0] += int(b.lengths.astype(np.int64).sum())
            t0 = time.perf_counter()
            E.run(rg, starts_all[off:off + n], rapp, eng, seed=0, sink=sink)
            return total[0], time.perf_counter() - t0
        return "reference", run, cores
    except ImportError:
        import oracle

        def run(n, off):
            t0 = time.perf_counter()
            _, ln, _ = oracle.walk(host_graph.offsets, host_graph.targets, host_graph.weights,
                                   host_graph.labels, starts_all[off:off + n], app=app.app,
                                   length=app.length, stop_prob=app.stop_prob, a=app.a,
                                   b=app.b, schema=app.schema, base_qid=off, threads=cores)
            return int(ln.astype(np.int64).sum()), time.perf_counter() - t0
        return "port", run, cores


def calibrate(run, seconds):
    """Warm the JIT, then size a sample to ~`seconds` of CPU work."""
    run(64, 0)
    n = 256
    while True:
        s, t = run(n, 0)
        if t > 1.0 or n >= 1 << 22:
            break
        n *= 4
    rate_q = n / max(t, 1e-6)
    return max(64, int(rate_q * seconds))


def cpu_baseline(host_graph, app, starts_all, seconds, sampler="auto"):
    kind, run, cores = reference_runner(host_graph, app, starts_all, sampler)
    n = min(calibrate(run, seconds), len(starts_all))
    sampled, t = run(n, 0)
    return {"value": sampled / t, "unit": "steps/s", "cores": cores, "kind": kind,
            "sample": f"{n} queries (global qids 0..{n - 1}) of the same workload, "
                      f"{sampled} sampled steps in {t:.1f} s, replay mode, workers={cores}"}


# ---------------------------------------------------------------------------
def make_starts(args, nv, hub):
    if args.queries == "hub":
        return np.full(nv, hub, np.int64)
    return np.arange(nv, dtype=np.int64)


def bench_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2404_08364_b200 import rmat
    app = app_config(args)
    g = rmat.rmat_graph(args.scale, labels=(args.app == "metapath"))
    if args.weights == "lognormal":
        from paper_2404_08364_b200.graph import synthesize_weights
        g = synthesize_weights(g, 2, "lognormal")
    starts = make_starts(args, g.vertex_count, g.max_degree_vertex())
    kind, run, cores = reference_runner(g, app, starts, args.sampler)
    n = min(calibrate(run, min(args.cpu_seconds, 8.0)), len(starts))
    for i in range(args.warmup):
        run(n, (i * n) % max(1, len(starts) - n))
    tot_s, tot_t = 0, 0.0
    for i in range(args.steps):
        s, t = run(n, ((args.warmup + i) * n) % max(1, len(starts) - n))
        tot_s += s
        tot_t += t
    value = tot_s / tot_t
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "fp64+u64", "data": "synthetic",
        "config": workload_config(args, app, int(os.environ.get("WORLD_SIZE", "1"))),
        "sample_queries_per_step": n,
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": kind,
                         "sample": f"{n} queries per step, replay mode, workers={cores}"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2404_08364_b200 as fw
    from paper_2404_08364_b200 import _lib, rmat
    from paper_2404_08364_b200.engine import DeviceGraph, _fw_structs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    # one GPU per rank over NCCL; with fewer GPUs than ranks (functional
    # testing on a 1-GPU box) the ranks share devices and talk over gloo
    backend = "nccl" if ndev >= world else "gloo"
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = dev if backend == "nccl" else torch.device("cpu")  # collective tensors
    if world > 1:
        if backend == "nccl":
            # communicator setup lines (nranks, NVLink/NVLS transport) for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    lib = _lib.load()
    app = app_config(args)
    labels = args.app == "metapath"

    # graph: generated on rank 0, replicated over NCCL (off the timed path)
    from paper_2404_08364_b200 import dist as fwd
    V = 1 << args.scale
    E_ = 16 * V
    if rank == 0:
        dg = rmat.rmat_graph_device(args.scale, labels=labels, device=local)
        if args.weights == "lognormal":  # synthesize_weights(g, 2, "lognormal") on the device copy
            w = np.random.default_rng(2).lognormal(0.0, 1.0, E_).astype(np.float32)
            wd = torch.empty(E_ + 4, dtype=torch.float32, device=dev)[:E_]  # 16-byte tail
            wd.copy_(torch.from_numpy(w))
            dg = DeviceGraph(V, E_, dg.offsets, dg.targets, wd, dg.labels, device=local)
            del w
        arrs = [dg.offsets, dg.targets, dg.weights] + ([dg.labels] if labels else [])
    if world > 1:
        sd = [(V + 1, torch.int64), (E_, torch.int32), (E_, torch.float32)] + \
            ([(E_, torch.uint8)] if labels else [])
        torch.cuda.synchronize()
        t_rep = time.perf_counter()
        if backend == "nccl":
            arrs = fwd.replicate_csr(arrs if rank == 0 else None, sd, src=0, device=dev)
        else:
            host = fwd.replicate_csr([t.cpu() for t in arrs] if rank == 0 else None, sd, src=0,
                                     device=cdev)
            if rank != 0:
                arrs = []
                for t, pad in zip(host, (0, 4, 4, 0)):
                    d = torch.empty(t.numel() + pad, dtype=t.dtype, device=dev)[:t.numel()]
                    d.copy_(t)
                    arrs.append(d)
        torch.cuda.synchronize()
        t_rep = time.perf_counter() - t_rep
        if rank != 0:
            dg = DeviceGraph(V, E_, *arrs[:3], arrs[3] if labels else None, device=local)
    handle = dg.handle(local).ptr
    hub = dg.max_degree_vertex()
    n_total = args.nq if args.nq else (V if args.scale < 26 else 1 << 24)
    if args.scaling == "strong":
        lo, hi = fwd.partition(n_total, world, rank)
    else:
        lo, hi = rank * n_total, (rank + 1) * n_total
    n = hi - lo
    base_qid = lo
    starts_h = (make_starts(args, V, hub)[np.arange(lo, hi) % V] if args.scaling == "strong"
                else make_starts(args, V, hub)[:n])
    starts = torch.from_numpy(np.ascontiguousarray(starts_h)).to(dev)
    L = app.length
    gather = ("none" if (args.no_gather or world == 1 or args.scaling != "strong")
              else args.gather)
    shared = None
    if gather == "direct":
        # rank 0's result buffers, exported by CUDA IPC: each rank's kernel
        # writes its qid range's rows straight into them (fused gather)
        own = None
        if rank == 0:
            own = [torch.empty(n_total * L, dtype=torch.int32, device=dev),
                   torch.empty(n_total, dtype=torch.int32, device=dev)]
        shared = fwd.share_buffers(own, src=0)
        seq_ptr = shared[0].data_ptr() + lo * L * 4
        len_ptr = shared[1].data_ptr() + lo * 4
    else:
        seq = torch.empty(n * L, dtype=torch.int32, device=dev)
        lens = torch.empty(n, dtype=torch.int32, device=dev)
        seq_ptr, len_ptr = seq.data_ptr(), lens.data_ptr()
    stats = torch.zeros(10, dtype=torch.int64, device=dev)
    a_s, e_s, _schema = _fw_structs(app, fw.EngineConfig(replay=True, sampler=args.sampler))
    stream = torch.cuda.current_stream(dev)

    def launch():
        stats[8:].zero_()  # per-launch first/last warp exit words
        _lib.check(lib.fw_walk_device(handle, starts.data_ptr(), n, base_qid, ctypes.byref(a_s),
                                      ctypes.byref(e_s), 0, seq_ptr, len_ptr,
                                      stats.data_ptr(), stream.cuda_stream))

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    stats.zero_()
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    ev[0].record(stream)
    for i in range(args.steps):
        launch()
        ev[i + 1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    launch_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    gather_ms = None
    if gather == "direct":
        # every rank's stores reached rank 0's buffer when its kernels
        # finished (synchronized above, then the barrier): no gather phase
        gather_ms = 0.0
        if args.dump_gather and rank == 0:  # consumed by tests/test_gpu_parity.py
            np.savez(args.dump_gather, seq=shared[0].view(n_total, L).cpu().numpy().view(np.uint32),
                     lens=shared[1].cpu().numpy().view(np.uint32))
    elif gather == "nccl":
        # rank 0 receives every other rank's segment (NCCL send/recv); the
        # time is the max over ranks of the device time around the exchange
        src_s, src_l = seq.to(cdev), lens.to(cdev)
        torch.cuda.synchronize()
        dist.barrier()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        t_g = time.perf_counter()
        g0.record()
        gathered = fwd.gather_paths(src_s, src_l, n_total, L, dst=0)
        g1.record()
        torch.cuda.synchronize()
        gm = torch.tensor([max(g0.elapsed_time(g1), 1000 * (time.perf_counter() - t_g))],
                          dtype=torch.float64, device=cdev)
        dist.all_reduce(gm, op=dist.ReduceOp.MAX)
        gather_ms = float(gm.item())
        if args.dump_gather and rank == 0:  # consumed by tests/test_gpu_parity.py
            np.savez(args.dump_gather, seq=gathered[0].cpu().numpy().view(np.uint32),
                     lens=gathered[1].cpu().numpy().view(np.uint32))
        del gathered, src_s, src_l
    my_ms = sum(launch_ms)
    st = stats.cpu().numpy()
    tail = {"last_launch_ms": launch_ms[-1],
            "tail_ms": (int(st[8]) - int(~np.uint64(st[9].view(np.uint64)))) * 1e-6,
            "note": "first to last warp exit in the last timed launch (%globaltimer)"}
    sampled = int(st[6])
    alg_bytes = int(st[7])
    t = torch.tensor([my_ms], dtype=torch.float64, device=cdev)
    tot = torch.tensor([sampled], dtype=torch.int64, device=cdev)
    per_rank_ms = [my_ms]
    if world > 1:
        allt = [torch.zeros(1, dtype=torch.float64, device=cdev) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank_ms = [float(x.item()) for x in allt]
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
    elapsed_ms = float(t.item())
    value = int(tot.item()) / (elapsed_ms / 1000.0)

    # end to end through the C ABI with pinned host buffers
    e2e = None
    summation = None
    if not args.no_e2e:
        hs = torch.from_numpy(starts_h).pin_memory()
        hseq = torch.empty(n * L, dtype=torch.int32).pin_memory()
        hlen = torch.empty(n, dtype=torch.int32).pin_memory()
        fst = _lib.FwStats()

        def host_call():
            _lib.check(lib.fw_walk(handle, hs.data_ptr(), n, base_qid, ctypes.byref(a_s),
                                   ctypes.byref(e_s), 0, hseq.data_ptr(), hlen.data_ptr(),
                                   ctypes.byref(fst)))
        host_call()
        host_call()
        # short launches (DeepWalk s16: 5 ms) are timed over >= 0.5 s of calls so
        # that one scheduling hiccup of the host thread does not set the figure
        e2e_iters = max(args.steps, int(math.ceil(0.5 / max(my_ms / args.steps / 1e3, 1e-6))))
        e2e_iters = min(e2e_iters, 1000)
        if world > 1:
            t_it = torch.tensor([e2e_iters], dtype=torch.int64, device=cdev)
            dist.all_reduce(t_it, op=dist.ReduceOp.MAX)
            e2e_iters = int(t_it.item())
            dist.barrier()
        t0 = time.perf_counter()
        e2e_sampled = 0
        call_ms, dev_ms = [], []
        for _ in range(e2e_iters):
            tc = time.perf_counter()
            host_call()
            call_ms.append(1e3 * (time.perf_counter() - tc))
            dev_ms.append(fst.total_ms)
            e2e_sampled += fst.sampled_steps
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=cdev)
        e2e_tot = torch.tensor([e2e_sampled], dtype=torch.int64, device=cdev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
            dist.all_reduce(e2e_tot, op=dist.ReduceOp.SUM)
        e2e = {"value": int(e2e_tot.item()) / float(e2e_s.item()), "unit": "steps/s",
               "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * L * 4 + n * 4,
               "path": "fw_walk (C ABI, pinned host buffers)", "iters": e2e_iters,
               "call_ms_median": statistics.median(call_ms),
               "device_ms_median": statistics.median(dev_ms),
               "d2h_pieces_overlapped": int(fst.d2h_pieces)}
        summation = {0: "sequential", 1: "exact", 2: "certified"}.get(int(fst.exact_order))
        del hseq

    peak, peak_kind = measured_peak()
    mean_launch_s = (my_ms / args.steps) / 1000.0
    achieved = (alg_bytes / args.steps) / mean_launch_s / 1e9
    workload = workload_name(args, app)
    traffic, traffic_basis = profiled_traffic(workload, alg_bytes / args.steps)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "peak_kind": peak_kind,
                "traffic": traffic, "traffic_basis": traffic_basis,
                "alg_bytes_per_launch": alg_bytes // args.steps,
                "kernel": "fw::walk_kernel (persistent, 1 launch per step)"}
    if traffic:
        # the measured DRAM rate next to the algorithmic one: frac counts the
        # bytes SURVEY 8(d) defines, much of which the walks re-read from L2
        roofline["dram_achieved"] = traffic / mean_launch_s / 1e9
        roofline["dram_frac"] = roofline["dram_achieved"] / peak
    counters = profiled_counters(workload)
    if counters:
        roofline["binding"] = ("issue: instruction issue, not HBM, limits this kernel "
                               "(DESIGN.md 3.3); DRAM and L2 run well below their peaks")
        roofline["counters"] = counters
    if roofline["frac"] > 1.0:
        roofline["note"] = ("algorithmic bytes exceed the HBM peak: the walks' adjacency is "
                            "L2-resident (re-read from the 126 MB L2), so frac is not an "
                            "HBM fraction here; see dram_frac and counters")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            host = dg.to_host()
            cpu = cpu_baseline(host, app, starts_h, args.cpu_seconds, args.sampler)
        except Exception as exc:  # report, never fail the GPU line
            cpu = {"value": None, "unit": "steps/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {type(exc).__name__}: {exc}"}

    if rank == 0:
        line = {
            "metric": metric_name(args), "value": value, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "fp64+u64", "data": "synthetic",
            "config": workload_config(args, app, world),
            "run": {"replicate_s": None if world == 1 else round(t_rep, 3),
                    "gather": gather, "gather_ms": gather_ms,
                    "gather_bytes": (n_total * L * 4 + n_total * 4) if gather != "none" else None,
                    "per_rank_walk_ms": [round(x, 3) for x in per_rank_ms],
                    "backend": backend if world > 1 else None, "summation": summation,
                    "sampled_steps_per_gpu_step": sampled // args.steps,
                    "walk_attempts_per_step": int(st[0]) // args.steps},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps, "load_imbalance_tail": tail,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if shared is not None:  # IPC views go before the exporting rank frees
            del shared
            torch.cuda.synchronize()
            dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
