"""Extra paths for compute-sanitizer beyond smoke(): evict_select's multi-round segments,
partitioned bucket levels and finish sorts (adversarial keys at 2^15), kv_truncate, the manager
step with device-resident chains, the fused-gather extra outputs, the uploaded-list path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_03651_b200 as K  # noqa: E402
import workloads as W  # noqa: E402

dev = "cuda"
rng = np.random.default_rng(0)
n = 1 << 15
cases = {
    "outliers": (np.where(rng.random(n) < 0.002, (1 << 60) + rng.integers(0, 1 << 30, n), 5).astype(np.uint64), n // 2),
    "take_all_skewed": (np.where(rng.random(n) < 0.1, rng.integers(1 << 50, 1 << 61, n), 1).astype(np.uint64), n + 3),
    "fin": (rng.integers(0, 1 << 20, n).astype(np.uint64), 777),
}
for name, (keys, k) in cases.items():
    ids, m = K.evict_select(torch.from_numpy(keys.view(np.int64)).to(dev), k)
    torch.cuda.synchronize()
    print(name, m)
wl = W.make_workload("tiny")
pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), K.free_bits_tensor(wl.free_bits, dev))
batch = K.Batch(wl.batch, dev)
K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
q = wl.q.to(dev)
out = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
extra = torch.empty_like(out)
plan = K.Plan(pool, batch)
plan.set_extra_outputs([extra])
plan.run(q, out)
keep = (wl.batch["ctx_len"] - np.diff(wl.batch["q_indptr"])).astype(np.int32)
K.kv_truncate(pool, batch, keep)
torch.cuda.synchronize()
assert torch.equal(out.view(torch.int16), extra.view(torch.int16))
ev = W.make_evict(n=1 << 14, k=1 << 10, seed=3)
t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).to(dev)  # noqa: E731
mgr = K.ManagerStep(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
chains = [(4, rng.choice(len(ev.state), 40, replace=False)), (2, rng.choice(len(ev.state), 25, replace=False))]
csr = K.ManagerStep.chains_to_device(K.ManagerStep.chains_csr(chains), dev)
mgr(5, csr, torch.from_numpy(rng.integers(0, len(ev.state), 300).astype(np.int32)).to(dev))
torch.cuda.synchronize()
# kv_manager_step_select (manager + selection in one kernel), twice on one workspace (the
# selection's cached layout), odd n (scalar slice tails)
n2 = len(ev.state) - 3
mgr2 = K.ManagerStep(t(ev.state[:n2], np.uint8), t(ev.rc[:n2], np.int32), t(ev.lat[:n2], np.int32),
                     t(ev.depth[:n2], np.int16))
sws = torch.empty(K.evict_select_workspace_size(n2, 1000), dtype=torch.uint8, device=dev)
sids = torch.empty(1000, dtype=torch.int32, device=dev)
for now in (6, 7):
    mgr2(now, chains, torch.from_numpy(rng.integers(0, n2, 300).astype(np.int32)).to(dev), select=(1000, sids, sws))
torch.cuda.synchronize()
# kv_append_plan (one call) on a fresh tiny workload
wl2 = W.make_workload("tiny")
pool2 = K.Pool(wl2.k_pool.to(dev), wl2.v_pool.to(dev), K.free_bits_tensor(wl2.free_bits, dev))
batch2 = K.Batch(wl2.batch, dev)
plan2 = K.kv_append_plan(pool2, batch2, wl2.k_new.to(dev), wl2.v_new.to(dev))
plan2.run(wl2.q.to(dev), torch.empty(wl2.q.shape, dtype=torch.bfloat16, device=dev))
torch.cuda.synchronize()
print("sanitize cases ok")
