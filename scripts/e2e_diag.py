"""Where the e2e time of a small fw_walk call goes (DeepWalk s16): wall time
vs device total (e0..e3) vs kernel, with and without the overlapped D2H."""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2404_08364_b200 as fw
from paper_2404_08364_b200 import _lib, rmat
from paper_2404_08364_b200.engine import _fw_structs

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
app = fw.AppConfig(app=sys.argv[2] if len(sys.argv) > 2 else "deepwalk", length=80)
lib = _lib.load()
dg = rmat.rmat_graph_device(scale, labels=False)
h = dg.handle(0).ptr
V = 1 << scale
a_s, e_s, _ = _fw_structs(app, fw.EngineConfig(replay=True))
hs = torch.arange(V, dtype=torch.int64).pin_memory()
hseq = torch.empty(V * 80, dtype=torch.int32).pin_memory()
hlen = torch.empty(V, dtype=torch.int32).pin_memory()
st = _lib.FwStats()
for label, env in (("overlap", {}), ("no-overlap", {"FW_D2H_OVERLAP": "0"})):
    os.environ.pop("FW_D2H_OVERLAP", None)
    os.environ.update(env)
    for _ in range(3):
        _lib.check(lib.fw_walk(h, hs.data_ptr(), V, 0, ctypes.byref(a_s), ctypes.byref(e_s), 0,
                               hseq.data_ptr(), hlen.data_ptr(), ctypes.byref(st)))
    walls, tots, kers = [], [], []
    for _ in range(10):
        t0 = time.perf_counter()
        _lib.check(lib.fw_walk(h, hs.data_ptr(), V, 0, ctypes.byref(a_s), ctypes.byref(e_s), 0,
                               hseq.data_ptr(), hlen.data_ptr(), ctypes.byref(st)))
        walls.append(1e3 * (time.perf_counter() - t0))
        tots.append(st.total_ms)
        kers.append(st.kernel_ms)
    print(f"{label}: wall {np.median(walls):.3f} ms, device total {np.median(tots):.3f} ms, "
          f"kernel {np.median(kers):.3f} ms, pieces {st.d2h_pieces}, steps/s wall "
          f"{st.sampled_steps / (np.median(walls) / 1e3):.4g}")
