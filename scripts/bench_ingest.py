"""Graph-ingest timing on one B200: the device
build_csr (fw_build_csr_device: stable LSD radix sort, lexsort semantics of
reswalk graph.py:138-169), the FWG1 load (fw_fwg1_read: 8 reader threads,
pinned double buffers, device CRC-32, graph.py:225-254) and fw_graph_create
from host arrays, at R-MAT scale 22 and 24.

Prints one JSON object per measurement.  The CPU column restates
build_csr's own numpy call (np.lexsort((dst, src)) + bincount) on the same
edges, timed on this host, for scale (it is the reference's algorithm, not
the oracle package).

    python scripts/bench_ingest.py [--scales 22 24] [--fwg1-dir /tmp]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--scales", type=int, nargs="+", default=[22, 24])
    p.add_argument("--fwg1-dir", default="/tmp")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cpu", action="store_true", help="also time numpy lexsort (slow at s24)")
    args = p.parse_args()

    import torch

    from paper_2404_08364_b200 import _lib, graph
    from paper_2404_08364_b200.rmat import GRAPH_SEED, RMAT_ABC

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    peak = None
    try:
        peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    for s in args.scales:
        V = 1 << s
        m = 8 * V
        E = 2 * m
        src = torch.empty(E, dtype=torch.int32, device=dev)
        dst = torch.empty(E, dtype=torch.int32, device=dev)
        _lib.check(lib.fw_rmat_edges_device(GRAPH_SEED, s, *RMAT_ABC, 0, m, src.data_ptr(),
                                            dst.data_ptr(), stream.cuda_stream))
        _lib.check(lib.fw_rmat_edges_device(GRAPH_SEED, s, *RMAT_ABC, 0, m,
                                            dst.data_ptr() + 4 * m, src.data_ptr() + 4 * m,
                                            stream.cuda_stream))
        off = torch.empty(V + 1, dtype=torch.int64, device=dev)
        tgt = torch.empty(E + 4, dtype=torch.int32, device=dev)[:E]
        w_in = torch.rand(E, device=dev, dtype=torch.float32)
        w_out = torch.empty(E + 4, dtype=torch.float32, device=dev)[:E]

        def build(with_w):
            _lib.check(lib.fw_build_csr_device(
                src.data_ptr(), dst.data_ptr(), w_in.data_ptr() if with_w else None, None, E, V,
                off.data_ptr(), tgt.data_ptr(), w_out.data_ptr() if with_w else None, None,
                stream.cuda_stream))

        for with_w in (False, True):
            build(with_w)  # warm-up (allocations)
            torch.cuda.synchronize()
            ms = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                build(with_w)
                e1.record(stream)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            best = min(ms)
            # algorithmic bytes: read the edge list once, write the CSR once
            alg = E * 8 + (V + 1) * 8 + E * 4 + (E * 8 if with_w else 0)
            line = {"what": "build_csr_device", "scale": s, "edges": E, "with_weights": with_w,
                    "ms": best, "edges_per_s": E / (best / 1e3),
                    "alg_bytes": alg, "alg_gbs": alg / (best / 1e3) / 1e9,
                    "hbm_peak_gbs": peak, "reps_ms": [round(x, 2) for x in ms]}
            print(json.dumps(line), flush=True)
        if args.cpu:
            hs, hd = src.cpu().numpy().view(np.uint32), dst.cpu().numpy().view(np.uint32)
            t0 = time.perf_counter()
            order = np.lexsort((hd, hs))
            targets = hd[order]
            offsets = np.zeros(V + 1, np.int64)
            np.cumsum(np.bincount(hs, minlength=V), out=offsets[1:])
            t = time.perf_counter() - t0
            ok = np.array_equal(targets, tgt.cpu().numpy().view(np.uint32)) and \
                np.array_equal(offsets, off.cpu().numpy())
            print(json.dumps({"what": "build_csr_numpy_lexsort (host, 1 thread)", "scale": s,
                              "edges": E, "s": t, "edges_per_s": E / t,
                              "equal_to_device": bool(ok)}), flush=True)
            del hs, hd, targets, order
        # FWG1: write once from the host, then stream it back to the device
        from paper_2404_08364_b200.engine import DeviceGraph
        dg = DeviceGraph(V, E, off, tgt, w_out, None, device=0)
        path = os.path.join(args.fwg1_dir, f"rmat{s}.fwg")
        hg = dg.to_host()
        graph.save_binary(hg, path)
        # fw_graph_create from host arrays (pinned-pool staged H2D + device CSR checks)
        import ctypes
        nbytes_h = hg.offsets.nbytes + hg.targets.nbytes + hg.weights.nbytes
        ts = []
        for _ in range(args.reps):
            off_, tgt_, w_ = hg.offsets, hg.targets, hg.weights
            out = ctypes.c_void_p()
            t0 = time.perf_counter()
            _lib.check(lib.fw_graph_create(off_.ctypes.data, tgt_.ctypes.data, w_.ctypes.data,
                                           None, V, E, 0, ctypes.byref(out)))
            ts.append(time.perf_counter() - t0)
            lib.fw_graph_destroy(out)
        print(json.dumps({"what": "fw_graph_create (host arrays -> HBM, incl. device CSR checks)",
                          "scale": s, "bytes": nbytes_h, "s": min(ts),
                          "gbs": nbytes_h / min(ts) / 1e9,
                          "reps_s": [round(x, 3) for x in ts]}), flush=True)
        del hg
        nbytes = os.path.getsize(path)
        ts = []
        for _ in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g2 = graph.load_binary_device(path)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            del g2
        print(json.dumps({"what": "load_binary_device (FWG1, CRC-32 on device)", "scale": s,
                          "file_bytes": nbytes, "s": min(ts), "gbs": nbytes / min(ts) / 1e9,
                          "note": "host file read (page cache after the first rep) + pinned H2D",
                          "reps_s": [round(x, 3) for x in ts]}), flush=True)
        os.unlink(path)
        buf = torch.randint(0, 255, (1 << 30,), dtype=torch.uint8, device=dev)
        out = np.zeros(1, np.uint32)
        _lib.check(lib.fw_crc32_device(buf.data_ptr(), buf.numel(), out.ctypes.data,
                                       stream.cuda_stream))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.reps):
            _lib.check(lib.fw_crc32_device(buf.data_ptr(), buf.numel(), out.ctypes.data,
                                           stream.cuda_stream))
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / args.reps
        print(json.dumps({"what": "crc32_device", "bytes": buf.numel(), "s": t,
                          "gbs": buf.numel() / t / 1e9}), flush=True)
        del src, dst, off, tgt, w_in, w_out, dg, buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
