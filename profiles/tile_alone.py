"""Tile-phase (tile_tc2_kernel) time alone for a config: median of N warm runs, CUDA events.
python profiles/tile_alone.py [config] [n]  -> one line: config, us, TFLOP/s (algorithmic)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "qwen14b-p"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
wl = W.make_workload(cfg, device=dev)
pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
batch = K.Batch(wl.batch, dev)
K.kv_append(pool, batch, wl.k_new, wl.v_new)
plan = K.Plan(pool, batch)
out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
s = torch.cuda.current_stream()
ts = []
for i in range(n + 3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    plan.run(wl.q, out, phases=K.PHASE_TILE)
    b.record(s)
    b.synchronize()
    if i >= 3:
        ts.append(a.elapsed_time(b) * 1e3)
us = statistics.median(ts)
print(f"{cfg} tile {us:.1f} us {plan.stats()['tile_flops'] / us / 1e6:.1f} TFLOP/s")
