"""Diagnostics: role timelines of tile_tc2_kernel's CTA 0 (option debug_ts: a device buffer).
Build with KVA_NVCC_DEFS=-DKVA_TILE_TIMESTAMPS (the stamps are compiled out by default)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
dev = torch.device("cuda", 0)
buf = torch.zeros(4 * 512, dtype=torch.int64, device=dev)
import numpy as np
import paper_2504_03651_b200 as K
import workloads as W
K.set_option("debug_ts", buf.data_ptr())
wl = W.make_workload(sys.argv[1] if len(sys.argv) > 1 else "llama7b", device=dev)
pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
batch = K.Batch(wl.batch, dev)
K.kv_append(pool, batch, wl.k_new, wl.v_new)
out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
plan = K.Plan(pool, batch)
for _ in range(3):
    buf.zero_()
    plan.run(wl.q, out, phases=K.PHASE_TILE)
torch.cuda.synchronize()
b = buf.cpu().numpy().reshape(4, 512)
t0 = b[b > 0].min()
res = {}
for r, name in enumerate(["mma", "sm0", "sm1", "prod"]):
    v = b[r][b[r] > 0] - t0
    res[name] = v[:120].tolist()
print(json.dumps(res))
