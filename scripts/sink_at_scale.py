"""Result sink at scale: run_batches over the s27 graph
with an Eq. 3 host memory budget that splits one query set into batches
(double-buffered: batch b+1 walks while the consumer holds batch b), and the
same queries in one device launch; the per-batch results must equal the
single launch's rows, and the FWR1 file written from the batches must read
back identically.  Prints one JSON line."""
import ctypes, json, os, sys, tempfile, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import _lib, rmat
from paper_2404_08364_b200.engine import _fw_structs

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
budget = int(float(sys.argv[3])) if len(sys.argv) > 3 else int(1.0e9)
t0 = time.perf_counter()
dg = rmat.rmat_graph_device(scale, labels=False)
gen_s = time.perf_counter() - t0
V = 1 << scale
rs = np.random.default_rng(7)
starts = rs.integers(0, V, nq).astype(np.int64)
app = fw.AppConfig(app="node2vec", length=80, a=2.0, b=0.5)
eng = fw.EngineConfig(replay=True, memory_budget=budget)
L = app.length
# reference rows: one device launch over the same qids
lib = _lib.load()
a_s, e_s, _ = _fw_structs(app, fw.EngineConfig(replay=True))
d_st = torch.from_numpy(starts).cuda()
d_seq = torch.empty(nq * L, dtype=torch.int32, device="cuda")
d_len = torch.empty(nq, dtype=torch.int32, device="cuda")
d_stats = torch.zeros(10, dtype=torch.int64, device="cuda")
_lib.check(lib.fw_walk_device(dg.handle(0).ptr, d_st.data_ptr(), nq, 0, ctypes.byref(a_s),
                              ctypes.byref(e_s), 0, d_seq.data_ptr(), d_len.data_ptr(),
                              d_stats.data_ptr(), None))
torch.cuda.synchronize()
ref_seq = d_seq.cpu().numpy().view(np.uint32).reshape(nq, L)
ref_len = d_len.cpu().numpy().view(np.uint32)
del d_seq, d_len
path = os.path.join(tempfile.gettempdir(), "sink_at_scale.fwr")
batches, mism = 0, 0
t1 = time.perf_counter()
chunks_s, chunks_l = [], []
for b in fw.run_batches(dg, starts, app, eng, seed=0):
    lo = b.base_qid
    mism += int(not np.array_equal(b.sequences, ref_seq[lo:lo + b.count]))
    mism += int(not np.array_equal(b.lengths, ref_len[lo:lo + b.count]))
    chunks_s.append(b.sequences.copy())
    chunks_l.append(b.lengths.copy())
    batches += 1
walk_s = time.perf_counter() - t1
del chunks_s, chunks_l
# FWR1 written batch by batch by the writer (engine.py:382-403 layout)
t2 = time.perf_counter()
fw.write_result_file(path, dg, starts, app, eng, seed=0)
fwr_s = time.perf_counter() - t2
rlen, rseq = fw.read_result_file(path)
fwr_ok = bool(np.array_equal(rseq, ref_seq) and np.array_equal(rlen, ref_len))
fwr_bytes = os.path.getsize(path)
os.unlink(path)
print(json.dumps({"scale": scale, "queries": nq, "memory_budget": budget,
                  "batch_size": fw.batch_size(eng, L), "batches": batches,
                  "batch_mismatches": mism, "fwr1_roundtrip_equal": fwr_ok,
                  "run_batches_s": walk_s, "fwr1_write_s": fwr_s, "fwr1_bytes": fwr_bytes, "sampled_steps": int(ref_len.astype(np.int64).sum()),
                  "graph_gen_s": gen_s}))
