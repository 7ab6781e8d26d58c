import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    """Reference-generated walk vectors (tests/golden/gen_golden.py)."""

    def __init__(self):
        with open(os.path.join(GOLDEN, "cases.json")) as fh:
            meta = json.load(fh)
        self.cases = {c["name"]: c for c in meta["cases"]}
        self.kats = meta["kats"]
        self.trials = meta.get("trials", [])
        self.z = np.load(os.path.join(GOLDEN, "walks.npz"))

    def graph(self, name):
        z = self.z
        lab = z.get(f"g_{name}_labels")
        return (z[f"g_{name}_offsets"], z[f"g_{name}_targets"], z[f"g_{name}_weights"], lab)

    def expected(self, name):
        z = self.z
        return (z[f"c_{name}_seq"], z[f"c_{name}_len"], z[f"c_{name}_stats"])

    def starts(self, name):
        return self.z[f"c_{name}_starts"]


@pytest.fixture(scope="session")
def golden():
    return Golden()


def case_kwargs(case):
    """Flatten a golden case into oracle.walk keyword arguments."""
    kw = dict(case["app"])
    if "schema" in kw:
        kw["schema"] = tuple(kw["schema"])
    eng = dict(case["eng"])
    for k in ("k_small", "k_big", "degree_threshold", "sampler"):
        if k in eng:
            kw[k] = eng[k]
    kw["seed"] = case["seed"]
    return kw, eng


def chi2_pass(counts, probs, alpha=1e-3):
    """Pearson chi-square of observed ``counts`` against exact ``probs``, with
    bins of expected count < 5 pooled (smallest first).  The reference's own
    gate is stats.passes_chi_square (stats.py:80-139)."""
    from scipy.stats import chi2
    counts = np.asarray(counts, dtype=np.float64)
    n = counts.sum()
    exp = np.asarray(probs, dtype=np.float64) * n
    order = np.argsort(exp, kind="stable")
    obs_p, exp_p, acc_o, acc_e = [], [], 0.0, 0.0
    for i in order:
        acc_o += counts[i]
        acc_e += exp[i]
        if acc_e >= 5:
            obs_p.append(acc_o)
            exp_p.append(acc_e)
            acc_o = acc_e = 0.0
    if acc_e > 0 and exp_p:
        obs_p[-1] += acc_o
        exp_p[-1] += acc_e
    obs_p, exp_p = np.array(obs_p), np.array(exp_p)
    stat = float(((obs_p - exp_p) ** 2 / exp_p).sum())
    dof = max(len(exp_p) - 1, 1)
    return stat <= chi2.ppf(1 - alpha, dof), stat, dof
