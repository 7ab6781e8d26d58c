"""Share of Node2Vec s22 lookups a dense-window bitmap could serve: sample
traversed edges (prev -> cur) uniformly, weight by d(cur), and count the window-path steps
whose N(prev) windows would fit a 47,104-bit bitmap."""
import numpy as np, sys
sys.path.insert(0,'/root/repo')
from paper_2404_08364_b200 import rmat
s=22
g=rmat.rmat_graph(s, labels=False)
off=g.offsets; deg=np.diff(off).astype(np.float64); V=len(deg)
E=len(g.targets)
rs=np.random.default_rng(0)
idx=rs.integers(0,E,3_000_000)
prev=np.searchsorted(off, idx, side='right')-1
cur=g.targets[idx].astype(np.int64)
dc=deg[cur]; dp=deg[prev]
W=dc.sum()
win = dp <= 4*dc+512
thr = 256*V/47104
dense = win & (dp >= thr)
print("V",V,"dense threshold dp >=",thr)
print("elements in window path", dc[win].sum()/W)
print("elements in dense-window steps", dc[dense].sum()/W)
print("steps dense", dense.mean())
