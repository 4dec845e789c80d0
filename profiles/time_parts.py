"""Per-call device timing of the hot-path pieces (CUDA events, warm, median of N).

python profiles/time_parts.py [config] — prints one JSON dict: kv_append, plan+run (all phases,
overlapped), tile-only, decode-only, merge-only, evict_keys, evict_select (1M, k=64k) in us.
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402


def timeit(fn, n=20, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(n):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "llama7b"
    dev = torch.device("cuda", 0)
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    pr_dev = batch.table_dev.clone()
    pr_host = batch.table_host.copy()
    mask = pr_host == -1
    ws = torch.empty(K.kv_append_workspace_size(batch), dtype=torch.uint8, device=dev)
    res = {}

    def app():
        batch.table_dev.copy_(pr_dev)
        batch.table_host[...] = pr_host
        K.kv_append(pool, batch, wl.k_new, wl.v_new, ws)
        K.kv_release_blocks(pool, batch.table_host[mask & (batch.table_host >= 0)])

    res["kv_append+release_us"] = timeit(app)
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        app()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res["kv_append+release_host_us_per_call"] = (t1 - t0) / 50 * 1e6
    app()
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    plan = K.Plan(pool, batch)
    res["attention_all_phases_us"] = timeit(lambda: plan.run(wl.q, out))
    res["tile_only_us"] = timeit(lambda: plan.run(wl.q, out, phases=K.PHASE_TILE))
    res["decode_only_us"] = timeit(lambda: plan.run(wl.q, out, phases=K.PHASE_DECODE))
    res["merge_only_us"] = timeit(lambda: plan.run(wl.q, out, phases=K.PHASE_MERGE))
    st = plan.stats()
    res["tile_tflops_alone"] = st["tile_flops"] / (res["tile_only_us"] * 1e-6) / 1e12
    res["decode_GBps_alone"] = st["decode_kv_bytes"] / (res["decode_only_us"] * 1e-6) / 1e9
    res["plan_stats"] = st
    ev = W.make_evict()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)
    stt, rc, lat, dep = t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16)
    keys = torch.empty(len(ev.state), dtype=torch.int64, device=dev)
    res["evict_keys_us"] = timeit(lambda: K.evict_keys(stt, rc, lat, dep, keys=keys))
    ids = torch.empty(ev.k, dtype=torch.int32, device=dev)
    wse = torch.empty(K.evict_select_workspace_size(len(ev.state), ev.k), dtype=torch.uint8, device=dev)
    res["evict_select_us"] = timeit(lambda: K.evict_select(keys, ev.k, out_ids=ids, workspace=wse, sync=False))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        pl = K.Plan(pool, batch, plan.workspace)
        pl.run(wl.q, out)
        pl.close()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    res["plan+run_host_us_per_call"] = (t1 - t0) / 50 * 1e6
    res["plan+run_wall_us_per_call"] = (t2 - t0) / 50 * 1e6
    print(json.dumps(res))




def evict_phases():
    """Phase timestamps (ns) of evict_select's CTA 0 (SelWs.t at workspace offset 256)."""
    dev = torch.device("cuda", 0)
    ev = W.make_evict()
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)
    keys = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
    wse = torch.zeros(K.evict_select_workspace_size(len(ev.state), ev.k), dtype=torch.uint8, device=dev)
    for _ in range(3):
        K.evict_select(keys, ev.k, workspace=wse)
    ts = wse[256:256 + 256].view(torch.int64).cpu().numpy()
    ts = ts[ts > 0]
    print(json.dumps({"evict_phase_ns": (ts - ts[0]).tolist()}))


def host_costs(cfg="llama7b"):
    """Host-side cost of each per-step API call (GPU drained before each call so that no
    staging wait is included)."""
    import time
    dev = torch.device("cuda", 0)
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = K.Batch(wl.batch, dev)
    pr_dev, pr_host = batch.table_dev.clone(), batch.table_host.copy()
    mask = pr_host == -1
    ws = torch.empty(K.kv_append_workspace_size(batch), dtype=torch.uint8, device=dev)
    wsa = torch.empty(K.hybrid_attention_workspace_size(batch), dtype=torch.uint8, device=dev)
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    acc = {}

    def t(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        acc.setdefault(name, []).append((time.perf_counter() - t0) * 1e6)
        return r
    for _ in range(20):
        t("table_reset", lambda: (batch.table_dev.copy_(pr_dev), batch.table_host.__setitem__(Ellipsis, pr_host)))
        t("kv_append", lambda: K.kv_append(pool, batch, wl.k_new, wl.v_new, ws))
        pl = t("plan", lambda: K.Plan(pool, batch, wsa))
        t("run", lambda: pl.run(wl.q, out))
        st = pl.stats()
        for k in ("host_validate_ns", "host_build_ns", "host_total_ns"):
            acc.setdefault("c++_" + k, []).append(st[k] / 1e3)
        t("release", lambda: K.kv_release_blocks(pool, batch.table_host[mask & (batch.table_host >= 0)]))
        t("plan_close", lambda: pl.close())
    print(json.dumps({k: round(statistics.median(v), 1) for k, v in acc.items()}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "evict":
        evict_phases()
    elif len(sys.argv) > 1 and sys.argv[1] == "host":
        host_costs(sys.argv[2] if len(sys.argv) > 2 else "llama7b")
    else:
        main()
