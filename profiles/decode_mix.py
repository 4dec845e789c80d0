"""decode_kt_kernel alone on qwen14b and its two halves (online decodes only / offline suffix
members only): GB/s of each, to locate the in-step inefficiency (short suffix units vs mix)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_03651_b200 as K
import workloads as W
from bench import _post_append_batch
dev = torch.device("cuda", 0)

def run(cfg):
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = _post_append_batch(K, wl, dev)
    plan = K.Plan(pool, batch)
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    plan.run(wl.q, out)
    for _ in range(3):
        plan.run(wl.q, out, phases=K.PHASE_DECODE)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        plan.run(wl.q, out, phases=K.PHASE_DECODE)
    b.record(); b.synchronize()
    ms = a.elapsed_time(b) / 20
    st = plan.stats()
    return {"config": cfg.name if hasattr(cfg, "name") else cfg, "decode_us": ms * 1e3,
            "GBps": st["decode_kv_bytes"] / (ms * 1e-3) / 1e9, "units": st["n_decode_items"]}

base = W.get_config("qwen14b")
if "--members-only" in sys.argv:  # for ncu: one members-only plan, decode phase
    members = [r for r in base.reqs if r.type != W.ONLINE_DECODE]
    run(W.custom_config("q-members", base.Hq, base.Hkv, base.d, 2, members, base.group_prefix_blocks))
    sys.exit(0)
online = [r for r in base.reqs if r.type == W.ONLINE_DECODE]
members = [r for r in base.reqs if r.type != W.ONLINE_DECODE]
print(json.dumps(run("qwen14b")))
print(json.dumps(run(W.custom_config("q-online", base.Hq, base.Hkv, base.d, 2, online, []))))
print(json.dumps(run(W.custom_config("q-members", base.Hq, base.Hkv, base.d, 2, members, base.group_prefix_blocks))))
print(json.dumps(run(W.custom_config("q-members-u", base.Hq, base.Hkv, base.d, 2,
      [W.ReqSpec(r.type, r.ctx, r.q_len, -1) for r in members], []))))
