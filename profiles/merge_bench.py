"""merge_kernel alone (phase KVA_PHASE_MERGE of a built plan), 50 back-to-back launches between
two CUDA events; the partials come from one full run of the same plan.

python profiles/merge_bench.py [config ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402
from bench import _post_append_batch  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in sys.argv[1:] or ["qwen14b", "llama7b"]:
    wl = W.make_workload(cfg, device=dev)
    pool = K.Pool(wl.k_pool, wl.v_pool, K.free_bits_tensor(wl.free_bits, dev))
    batch = _post_append_batch(K, wl, dev)
    plan = K.Plan(pool, batch)
    out = torch.empty(wl.q.shape, dtype=torch.bfloat16, device=dev)
    plan.run(wl.q, out)
    for _ in range(5):
        plan.run(wl.q, out, phases=K.PHASE_MERGE)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        plan.run(wl.q, out, phases=K.PHASE_MERGE)
    b.record()
    b.synchronize()
    st = plan.stats()
    print(json.dumps({"config": cfg, "merge_us": a.elapsed_time(b) * 1e3 / 50, "merge_rows": st["n_merge_rows"]}))
