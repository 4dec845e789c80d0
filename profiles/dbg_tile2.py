import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import workloads as W
from gpu_util import gpu_step, oracle_step
cases = {
  "one_chunk_64keys": (64, 1, 1, [W.ReqSpec(W.OFFLINE_PREFILL, 64, 64, -1)]),
  "one_chunk_128": (64, 1, 1, [W.ReqSpec(W.OFFLINE_PREFILL, 128, 128, -1)]),
  "one_chunk_200": (64, 1, 1, [W.ReqSpec(W.OFFLINE_PREFILL, 200, 200, -1)]),
  "prefix_chunk": (64, 1, 1, [W.ReqSpec(W.OFFLINE_PREFILL, 300, 100, -1)]),
  "d128_chunk_200": (128, 1, 1, [W.ReqSpec(W.OFFLINE_PREFILL, 200, 200, -1)]),
}
which = sys.argv[1:] or list(cases)
for name in which:
    d, g, Hkv, reqs = cases[name]
    wl = W.make_workload(W.custom_config(name, g * Hkv, Hkv, d, 3, reqs, []))
    gg = gpu_step(wl)
    r = oracle_step(wl)
    o = gg["out"].float().cpu().numpy().astype(np.float64)
    e = np.abs(o - r["out"]).max(axis=(1, 2))
    bad = np.nonzero(e > 1e-2)[0]
    print(name, "max err %.3e" % e.max(), "bad rows", bad[:10], len(bad), flush=True)
