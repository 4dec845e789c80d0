"""GPU parity of the alternative tile-kernel implementations and launch modes, each in a fresh
process (the implementation is chosen once per process from KVA_TILE_IMPL / KVA_OVERLAP /
KVA_TILE_CTAS): legacy mma.sync (64-row tiles), tcgen05 one-Q-tile, tcgen05 two-Q-tile
(default), tcgen05 CTA-pair (cta_group::2), and overlapped vs sequential scheduling; the two
decode kernels (v1: rows along M, v2: keys along M) and v2's two occupancy configurations; the
tile kernel's exp2 split between MUFU and the FMA-pipe polynomial (KVA_POLY pairs of 16)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import workloads as W
from gpu_util import gpu_step, oracle_step, assert_attention_close
reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 600 + 300, 300, 0), W.ReqSpec(W.OFFLINE_PREFILL, 600 + 173, 173, 0),
        W.ReqSpec(W.ONLINE_DECODE, 2000, 1), W.ReqSpec(W.ONLINE_DECODE, 77, 1)]
reqs += [W.ReqSpec(W.OFFLINE_DECODE, 600 + 5 + i, 1, 0) for i in range(20)]
reqs += [W.ReqSpec(W.OFFLINE_DECODE, 1100, 2), W.ReqSpec(W.OFFLINE_DECODE, 730, 2, 0)]
for d, Hq, Hkv in [(128, 16, 2), (64, 8, 4)]:
    wl = W.make_workload(W.custom_config("v", Hq, Hkv, d, 7, reqs, [600 // 16]))
    g = gpu_step(wl)
    r = oracle_step(wl)
    assert_attention_close(g["out"], g["lse"], r["out"], r["lse"])
    np.save({out!r} + f"_{{d}}.npy", g["out"].cpu().numpy())
print("OK")
'''


def _run(env_extra, tag, tmp_path):
    out = str(tmp_path / tag)
    env = dict(os.environ, **env_extra)
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
    return out


@pytest.mark.parametrize("impl", ["mma", "tc1", "tc2", "tc3"])
def test_tile_impl_parity(impl, tmp_path):
    _run({"KVA_TILE_IMPL": impl}, impl, tmp_path)


def test_overlap_modes_bitexact(tmp_path):
    import numpy as np
    a = _run({"KVA_OVERLAP": "1", "KVA_TILE_CTAS": "40"}, "ov", tmp_path)
    b = _run({"KVA_OVERLAP": "0"}, "seq", tmp_path)
    for d in (128, 64):
        assert np.array_equal(np.load(a + f"_{d}.npy"), np.load(b + f"_{d}.npy"))


@pytest.mark.parametrize("env", [{"KVA_DECODE_IMPL": "v1"}, {"KVA_DECODE_CFG": "1"},
                                 {"KVA_POLY": "0"}, {"KVA_POLY": "4"}, {"KVA_PDL": "0"}, {"KVA_TMA3D": "0"},
                                 {"KVA_TILE_K3": "0"}])
def test_decode_impl_parity(env, tmp_path):
    _run(env, "dec_" + "_".join(env.values()), tmp_path)


@pytest.mark.parametrize("ctas", ["1", "7", "148", "296"])
def test_evict_select_grid_sizes(ctas):
    """The selection's per-CTA bin reservations and segment ranges give the oracle's eviction
    order for any cooperative grid size (KVA_EVICT_CTAS), on the full-size `evict` config, its
    straddle variant and a skewed adversarial case."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, workloads as W, paper_2504_03651_b200 as K
for straddle in (False, True):
    ev = W.make_evict(straddle=straddle)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()
    keys = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
    ids, n = K.evict_select(keys, ev.k)
    _, rk = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    _, rids = oracle.evict_select(rk, ev.k)
    assert np.array_equal(ids.cpu().numpy(), rids), straddle
rng = np.random.default_rng(5)
keys = np.full(1 << 16, 5, np.uint64)
keys[rng.choice(1 << 16, 50, replace=False)] = np.uint64(1 << 61)
ids, n = K.evict_select(torch.from_numpy(keys.view(np.int64)).cuda(), 40000)
_, rids = oracle.evict_select(keys, 40000)
assert np.array_equal(ids.cpu().numpy(), rids)
print("OK")
""" % ROOT
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, KVA_EVICT_CTAS=ctas),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_pdl_merge_waits_for_the_tile_kernel(tmp_path):
    """Under PDL the decode kernel may start (and finish) while the tile kernel still runs; the
    merge after it reads cascade partials the TILE kernel writes.  Force the tile kernel to be
    the long pole (1 persistent CTA, a long prefill chunk in the batch) with the workspace
    NaN-filled: a merge that did not wait for it would produce NaN / wrong rows."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import workloads as W, paper_2504_03651_b200 as K
from gpu_util import oracle_step, assert_attention_close
reqs = [W.ReqSpec(W.OFFLINE_DECODE, 40 * 16 + 3 + i, 1, 0) for i in range(12)]
reqs += [W.ReqSpec(W.OFFLINE_PREFILL, 40 * 16 + 1500, 1500, 0), W.ReqSpec(W.ONLINE_DECODE, 900, 1)]
wl = W.make_workload(W.custom_config("pdl", 16, 2, 128, 61, reqs, [40]))
dev = "cuda"
pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), K.free_bits_tensor(wl.free_bits, dev))
batch = K.Batch(wl.batch, dev)
K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
ws = torch.full((K.hybrid_attention_workspace_size(batch) // 4 + 64,), float("nan"), device=dev).view(torch.uint8)
plan = K.Plan(pool, batch, ws)
assert plan.stats()["n_cascade_items"] > 0
q = wl.q.to(dev)
out = torch.empty(q.shape, dtype=torch.float32, device=dev)
lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
plan.run(q, out, lse)
torch.cuda.synchronize()
r = oracle_step(wl)
assert_attention_close(out, lse, r["out"], r["lse"])
print("OK")
""" % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, KVA_TILE_CTAS="1", KVA_OVERLAP="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
