"""Host (enqueue) time of each call of the bench step, measured from Python with perf_counter
over many steps (median us): python profiles/host_calls.py [config]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen14b"
dev = torch.device("cuda", 0)
wl = W.make_workload(cfg, device=dev)
pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
batch = K.Batch(wl.batch, dev)
ws_app = torch.empty(K.kv_append_workspace_size(batch), dtype=torch.uint8, device=dev)
ws_att = torch.empty(K.hybrid_attention_workspace_size(batch), dtype=torch.uint8, device=dev)
q, k_new, v_new = wl.q.to(dev), wl.k_new.to(dev), wl.v_new.to(dev)
out = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
keep = (wl.batch["ctx_len"] - np.diff(wl.batch["q_indptr"])).astype(np.int32)
ev = W.make_evict()
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
mgr = K.ManagerStep(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
chains, pool_chains = W.make_manager_update(ev, now=1 << 20, seed=1)
csr = K.ManagerStep.chains_to_device(K.ManagerStep.chains_csr(chains), dev)
pids = torch.from_numpy(np.concatenate(pool_chains[:1000]).astype(np.int32)).to(dev)
sel_ws = torch.empty(K.evict_select_workspace_size(len(ev.state), ev.k), dtype=torch.uint8, device=dev)
sel_ids = torch.empty(ev.k, dtype=torch.int32, device=dev)
s = torch.cuda.current_stream()
side = torch.cuda.Stream()
T = {k: [] for k in ("mgr_select", "kv_append_plan", "run", "truncate", "close")}
for it in range(300):
    a = time.perf_counter()
    mgr(1 << 20, csr, pids, recount=False, stream=side, select=(ev.k, sel_ids, sel_ws))
    b = time.perf_counter()
    plan = K.kv_append_plan(pool, batch, k_new, v_new, ws_app, ws_att, stream=s)
    c = time.perf_counter()
    plan.run(q, out, lse, stream=s)
    d = time.perf_counter()
    K.kv_truncate(pool, batch, keep, stream=s)
    e = time.perf_counter()
    plan.close()
    f = time.perf_counter()
    if it >= 20:
        for k, v in zip(T, (b - a, c - b, d - c, e - d, f - e)):
            T[k].append(v * 1e6)
    if it % 50 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
print({k: round(statistics.median(v), 1) for k, v in T.items()}, "total", round(sum(statistics.median(v) for v in T.values()), 1))
