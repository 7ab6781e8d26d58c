"""Sampler trials on the GPU: API twin of reswalk.trials.run_trials
(trials.py:46-90) over the sm_100a trial kernels (csrc/fw_trials.cu).

Trial t draws from the streams (t << 10) | lane, so picks, collective counts
and rejection rounds are bit-identical to the reference's numba kernels
(_kernels.py:84-277).  The timer covers only the device sampling launch
(CUDA events), like the reference's covers only its sampling loop.
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ValidationError

SAMPLERS = ("seq", "dprs", "zprs", "its", "alias", "rjs")
LANE_SAMPLERS = ("dprs", "zprs")
_METHOD = {"seq": 0, "dprs": 1, "zprs": 2, "its": 3, "alias": 4, "rjs": 5, "uniform-control": 6}


@dataclass
class TrialResult:
    sampler: str
    k: int
    n: int
    trials: int
    picks: np.ndarray
    elapsed_ns: int
    collectives_per_task: float
    collectives: np.ndarray | None = None
    rounds: np.ndarray | None = None


def alias_table(w):
    """Two-array alias table built exactly as samplers.alias_build
    (samplers.py:245-266): buckets scaled by n/total, small/large stacks
    popped from the end, leftovers pinned to probability 1."""
    w = np.asarray(w, dtype=np.float64)
    n = len(w)
    total = w.sum()
    if n == 0 or total <= 0.0:
        raise ValidationError("alias table needs positive total weight")
    prob = w * (n / total)
    alias = np.arange(1, n + 1, dtype=np.int64)
    small = [i for i in range(n) if prob[i] < 1.0]
    large = [i for i in range(n) if prob[i] >= 1.0]
    while small and large:
        s_i = small.pop()
        g_i = large.pop()
        alias[s_i] = g_i + 1
        prob[g_i] -= 1.0 - prob[s_i]
        (small if prob[g_i] < 1.0 else large).append(g_i)
    for i in large + small:
        prob[i] = 1.0
    return prob, alias


def run_trials(sampler, weights, trials, seed, k=32, max_rounds=10_000, device=0):
    """Run one (sampler, weights, k) cell on the GPU; same result fields as
    the reference's run_trials."""
    import ctypes

    import torch

    w = np.ascontiguousarray(weights, dtype=np.float64)
    if np.any(np.isnan(w)) or np.any(w < 0):
        raise ValidationError("weights must be non-negative and not NaN")
    if sampler not in _METHOD:
        raise ValidationError(f"unknown sampler {sampler!r}")
    lib = _lib.load()
    _lib.require_device()
    dev = torch.device("cuda", device)
    n = len(w)
    dw = torch.from_numpy(w if n else np.zeros(1)).to(dev)
    prob = alias = None
    if sampler == "alias":
        p, al = alias_table(w)
        prob, alias = torch.from_numpy(p).to(dev), torch.from_numpy(al).to(dev)
    w_max = float(w.max()) if n else 0.0
    picks = torch.empty(max(trials, 1), dtype=torch.int32, device=dev)
    aux = torch.empty(max(trials, 1), dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.check(lib.fw_sampler_trials_device(
            _METHOD[sampler], dw.data_ptr(), n, k, seed & 0xFFFFFFFFFFFFFFFF, trials,
            None if prob is None else prob.data_ptr(),
            None if alias is None else alias.data_ptr(), w_max, max_rounds,
            picks.data_ptr(), aux.data_ptr(), ctypes.c_void_p(stream.cuda_stream)))
        e1.record(stream)
        torch.cuda.synchronize(dev)
    elapsed = int(e0.elapsed_time(e1) * 1e6)
    picks_h = picks[:trials].cpu().numpy().view(np.uint32)
    aux_h = aux[:trials].cpu().numpy()
    collectives = aux_h if sampler in LANE_SAMPLERS else None
    rounds = aux_h if sampler == "rjs" else None
    per_task = float(collectives.mean()) if collectives is not None and trials else 0.0
    return TrialResult(sampler=sampler, k=k, n=n, trials=trials, picks=picks_h,
                       elapsed_ns=elapsed, collectives_per_task=per_task,
                       collectives=collectives, rounds=rounds)
