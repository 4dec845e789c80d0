"""Debug: per-request max error of the GPU path vs the oracle on the random mixed batches."""
import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import workloads as W
from gpu_util import gpu_step, oracle_step
from test_gpu_parity import _rand_cfg
for seed, d, g, Hkv in [(2, 64, 4, 2), (1, 128, 1, 2), (3, 128, 5, 2)]:
    wl = W.make_workload(_rand_cfg(seed, d, g, Hkv, nreq=9))
    gg = gpu_step(wl)
    r = oracle_step(wl)
    o = gg["out"].float().cpu().numpy().astype(np.float64)
    qi = wl.batch["q_indptr"]
    ql = np.diff(qi)
    print("cfg", seed, d, g, Hkv, "max err", np.nanmax(np.abs(o - r["out"])), "nan", np.isnan(o).sum())
    for i in range(len(ql)):
        e = np.abs(o[qi[i]:qi[i+1]] - r["out"][qi[i]:qi[i+1]])
        print("  req", i, "type", wl.batch["req_type"][i], "ql", ql[i], "ctx", wl.batch["ctx_len"][i], "grp", wl.batch["group_of"][i] if wl.batch.get("group_of") is not None else None, "err %.3e" % np.nanmax(e), "nan", int(np.isnan(e).sum()))
