"""The public Python API end to end (run() with a sink, host starts, host
results) against the C-ABI e2e for the headline workload."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dg = rmat.rmat_graph_device(scale, labels=False)
starts = np.arange(1 << scale, dtype=np.int64)
app = fw.AppConfig(app="node2vec", length=80, a=2.0, b=0.5)
eng = fw.EngineConfig(replay=True)
tot = [0]
def sink(b):
    tot[0] += int(b.lengths.sum())
fw.run(dg, starts, app, eng, seed=0, sink=sink)
for rep in range(3):
    tot[0] = 0
    t0 = time.perf_counter()
    st = fw.run(dg, starts, app, eng, seed=0, sink=sink)
    t = time.perf_counter() - t0
    print(f"run(): {tot[0] / t:.4g} sampled steps/s (wall {t:.3f} s, kernel {st.kernel_ms:.1f} ms)")
