"""Host-side (enqueue) cost of each call of one bench step, in us (perf_counter; the device is
synchronised before each call so nothing queues behind GPU work).

python profiles/host_parts.py [config]
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "llama7b"
    dev = torch.device("cuda", 0)
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    pr_dev, pr_host = batch.table_dev.clone(), batch.table_host.copy()
    mask = pr_host == -1
    ws_app = torch.empty(K.kv_append_workspace_size(batch), dtype=torch.uint8, device=dev)
    ws_att = torch.empty(K.hybrid_attention_workspace_size(batch), dtype=torch.uint8, device=dev)
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(wl.q.shape[:2], dtype=torch.float32, device=dev)
    evw = W.make_evict()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)
    st, rc, lat, dp = t(evw.state, np.uint8), t(evw.rc, np.int32), t(evw.lat, np.int32), t(evw.depth, np.int16)
    chains, mpool = W.make_manager_update(evw, now=1 << 20, seed=1)
    mgr = K.ManagerStep(st, rc, lat, dp)
    csr = K.ManagerStep.chains_csr(chains)
    rng = np.random.default_rng(11)
    moved = [mpool[i] for i in rng.choice(len(mpool), len(mpool) // 100, replace=False)]
    pids = torch.from_numpy(np.concatenate(moved).astype(np.int32)).to(dev)
    ids = torch.empty(evw.k, dtype=torch.int32, device=dev)
    wse = torch.empty(K.evict_select_workspace_size(len(evw.state), evw.k), dtype=torch.uint8, device=dev)
    parts = {}

    def tm(name, fn):
        torch.cuda.synchronize()
        a = time.perf_counter()
        r = fn()
        parts.setdefault(name, []).append((time.perf_counter() - a) * 1e6)
        return r

    for it in range(30):
        tm("manager_step", lambda: mgr(1 << 20, csr, pids, del_ids=pids, recount=False))
        tm("evict_select", lambda: K.evict_select(mgr.keys, evw.k, out_ids=ids, workspace=wse, sync=False))
        tm("table_reset", lambda: (batch.table_dev.copy_(pr_dev, non_blocking=True),
                                   batch.table_host.__setitem__(Ellipsis, pr_host)))
        tm("kv_append", lambda: K.kv_append(pool, batch, wl.k_new, wl.v_new, ws_app))
        plan = tm("plan", lambda: K.Plan(pool, batch, ws_att))
        tm("run", lambda: plan.run(wl.q, out, lse))
        alloc = batch.table_host[mask & (batch.table_host >= 0)]
        tm("release", lambda: K.kv_release_blocks(pool, alloc))
        tm("plan_close", lambda: plan.close())
    res = {k: round(statistics.median(v[5:]), 1) for k, v in parts.items()}
    res["total"] = round(sum(res.values()), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
