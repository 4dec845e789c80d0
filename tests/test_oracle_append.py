"""Pins for the kv_append + allocation oracle (Eq.(5)).

* Brute force: a sequential Python loop that walks requests in descriptor order and
  positions ascending and takes the smallest free id (reading #13) -> tables bit-exact.
* Definition: the pool after append equals the pool before with exactly the addressed
  slots overwritten; gathering through the table returns the written rows; NaN poison
  survives everywhere else.
* Atomicity of NEEDS_EVICTION and the capacity error.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W


def _free_list(bits, n):
    return [b for b in range(n) if (int(bits[b // 32]) >> (b % 32)) & 1]


def _brute_tables(b, bits):
    bt = b["block_table"].copy()
    free = _free_list(bits, b["num_blocks"])
    for i in range(b["num_reqs"]):
        ql = b["q_indptr"][i + 1] - b["q_indptr"][i]
        ctx = int(b["ctx_len"][i])
        for t in range(ctx - ql, ctx):
            if bt[i, t // 16] == -1:
                bt[i, t // 16] = free.pop(0)
    return bt, free


@pytest.mark.parametrize("name", ["tiny", "rand1", "rand2"])
def test_append_bruteforce_and_definition(name):
    if name == "tiny":
        wl = W.make_workload("tiny")
    else:
        rng = np.random.default_rng(len(name) + int(name[-1]))
        reqs = []
        for _ in range(5):
            ctx = int(rng.integers(1, 200))
            ql = int(rng.integers(1, ctx + 1))
            reqs.append(W.ReqSpec(W.OFFLINE_PREFILL, ctx, ql))
        wl = W.make_workload(W.custom_config(name, 2, 2, 64, int(name[-1]), reqs, []))
    b = wl.batch
    st, deficit, kp, vp, bt, fb = oracle.kv_append(b, wl.k_pool, wl.v_pool, wl.free_bits,
                                                  wl.k_new, wl.v_new)
    assert st == oracle.OK and deficit == 0
    exp_bt, exp_free = _brute_tables(b, wl.free_bits)
    assert np.array_equal(bt, exp_bt)
    assert _free_list(fb, b["num_blocks"]) == exp_free
    # definition: addressed slots overwritten with the new rows, everything else unchanged
    before_k = wl.k_pool.view(torch.int16).numpy().view(np.uint16)
    before_v = wl.v_pool.view(torch.int16).numpy().view(np.uint16)
    kn = wl.k_new.view(torch.int16).numpy().view(np.uint16)
    vn = wl.v_new.view(torch.int16).numpy().view(np.uint16)
    exp_k, exp_v = before_k.copy(), before_v.copy()
    for i in range(b["num_reqs"]):
        q0, q1 = b["q_indptr"][i], b["q_indptr"][i + 1]
        ctx = int(b["ctx_len"][i])
        for j in range(q1 - q0):
            t = ctx - (q1 - q0) + j
            exp_k[exp_bt[i, t // 16], :, t % 16] = kn[q0 + j]
            exp_v[exp_bt[i, t // 16], :, t % 16] = vn[q0 + j]
    assert np.array_equal(kp, exp_k) and np.array_equal(vp, exp_v)
    # every position [0, ctx) is now finite; unwritten slots stay NaN (0x7fc0 poison)
    written = np.zeros(kp.shape[:1] + kp.shape[2:3], bool)  # [blocks][16]
    for i in range(b["num_reqs"]):
        for t in range(int(b["ctx_len"][i])):
            written[bt[i, t // 16], t % 16] = True
    kf = torch.from_numpy(kp.view(np.int16)).view(torch.bfloat16).float()
    wmask = torch.from_numpy(written)
    assert torch.isfinite(kf.permute(0, 2, 1, 3)[wmask]).all()
    assert torch.isnan(kf.permute(0, 2, 1, 3)[~wmask]).all()


def test_partial_block_is_filled_first():
    cfg = W.custom_config("pb", 1, 1, 64, 3, [W.ReqSpec(W.ONLINE_DECODE, 21, 3)], [])
    wl = W.make_workload(cfg)
    b = wl.batch
    st, _, _, _, bt, _ = oracle.kv_append(b, wl.k_pool, wl.v_pool, wl.free_bits, wl.k_new, wl.v_new)
    assert st == oracle.OK
    # resident [0,18): block 1 is the partial block holding 16,17 and is reused for 18..20
    assert b["block_table"][0, 1] >= 0 and bt[0, 1] == b["block_table"][0, 1]
    assert np.array_equal(bt, b["block_table"])  # no new block allocated


def test_needs_eviction_is_atomic():
    wl = W.make_workload("tiny")
    b = wl.batch
    bits = wl.free_bits.copy()
    free = _free_list(bits, b["num_blocks"])
    need = 6 * 4  # tiny: 6 chunks x 4 new blocks
    for blk in free[: len(free) - (need - 5)]:   # leave need-5 free blocks
        bits[blk // 32] &= ~np.uint32(1 << (blk % 32))
    st, deficit, kp, vp, bt, fb = oracle.kv_append(b, wl.k_pool, wl.v_pool, bits, wl.k_new, wl.v_new)
    assert st == oracle.NEEDS_EVICTION and deficit == 5
    assert np.array_equal(bt, b["block_table"]) and np.array_equal(fb, bits)
    assert np.array_equal(kp, wl.k_pool.view(torch.int16).numpy().view(np.uint16))


def test_capacity_and_invalid():
    cfg = W.custom_config("cap", 1, 1, 64, 3, [W.ReqSpec(W.OFFLINE_PREFILL, 200, 200)], [])
    w2 = W.make_workload(cfg)
    b = dict(w2.batch)
    b["num_blocks"] = 10   # a 200-token request needs 13 blocks: UnsatisfiableAllocation
    st, *_ = oracle.kv_append(b, w2.k_pool, w2.v_pool, w2.free_bits, w2.k_new, w2.v_new)
    assert st == oracle.CAPACITY
    wl = W.make_workload("tiny")
    b = dict(wl.batch)
    bt = b["block_table"].copy()
    bt[0, 3] = -1          # a resident position without a block
    b["block_table"] = bt
    st, *_ = oracle.kv_append(b, wl.k_pool, wl.v_pool, wl.free_bits, wl.k_new, wl.v_new)
    assert st == oracle.INVALID
