import os, sys, time, statistics
sys.path.insert(0, '.')
import torch
import paper_2504_03651_b200 as K, workloads as W
from bench import _post_append_batch
dev = torch.device("cuda", 0)
wl = W.make_workload("llama7b", device=dev)
pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
batch = _post_append_batch(K, wl, dev)
plan = K.Plan(pool, batch)
out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
for ph, name in [(K.PHASE_DECODE, "decode 14KB"), (K.PHASE_MERGE, "merge 27KB"), (K.PHASE_TILE, "tile 22KB")]:
    ts = []
    for i in range(40):
        torch.cuda.synchronize()
        a = time.perf_counter(); plan.run(wl.q, out, phases=ph); ts.append((time.perf_counter() - a) * 1e6)
    print(name, round(statistics.median(ts[5:]), 1), "us host")
x = torch.empty(1, device=dev)
ts = []
for i in range(40):
    torch.cuda.synchronize(); a = time.perf_counter(); x.add_(1); ts.append((time.perf_counter() - a) * 1e6)
print("torch add_", round(statistics.median(ts[5:]), 1))
