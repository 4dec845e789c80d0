"""Pins for the attention oracle, all independent of the oracle's code.

Each test compares ``oracle.attention`` against something the paper or mathematics fixes:
the textbook definition written densely in numpy (unpaged, contiguous gather), a library
routine (torch SDPA fp64), closed forms, and invariants (paging, sharing, chunking, GQA).
A dropped scale, a wrong GQA map, an off-by-one causal limit, a transposed operand or a
wrong block lookup each fails at least one of them.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads as W


def _bf16_to_f64(t):
    return t.float().double().numpy()


def _post_state(wl):
    """All positions resident (generator's preappended mode): pools hold [0, ctx)."""
    return wl.batch, wl.k_pool, wl.v_pool, wl.q


def _gather_dense(b, pool, i, kvh):
    """Contiguous K (or V) rows [0, ctx) of request i, kv-head kvh, walked through the table."""
    ctx = int(b["ctx_len"][i])
    rows = []
    for t in range(ctx):
        blk = b["block_table"][i, t // 16]
        rows.append(pool[blk, kvh, t % 16])
    return np.stack(rows)


def _dense_reference(b, kp, vp, q):
    """softmax(Q K^T * s + offset-causal mask) V, unpaged, by the textbook definition."""
    kp, vp, qd = _bf16_to_f64(kp), _bf16_to_f64(vp), _bf16_to_f64(q)
    Hq, Hkv, d = b["num_q_heads"], b["num_kv_heads"], b["head_dim"]
    g = Hq // Hkv
    s = 1.0 / math.sqrt(d)
    out = np.zeros_like(qd)
    lse = np.zeros(qd.shape[:2])
    for i in range(b["num_reqs"]):
        q0, q1 = b["q_indptr"][i], b["q_indptr"][i + 1]
        ql, ctx = q1 - q0, int(b["ctx_len"][i])
        for h in range(Hq):
            K = _gather_dense(b, kp, i, h // g)
            V = _gather_dense(b, vp, i, h // g)
            Q = qd[q0:q1, h]
            S = (Q @ K.T) * s
            pos = np.arange(ctx - ql, ctx)[:, None]
            S = np.where(np.arange(ctx)[None, :] <= pos, S, -np.inf)
            m = S.max(axis=1, keepdims=True)
            P = np.exp(S - m)
            Z = P.sum(axis=1, keepdims=True)
            out[q0:q1, h] = (P @ V) / Z
            lse[q0:q1, h] = (m + np.log(Z))[:, 0]
    return out, lse


def _random_cfg(rng, d, g, Hkv=2, nreq=3, seed=0, with_group=False):
    reqs = []
    gp = []
    if with_group:
        gp = [int(rng.integers(1, 4))]
    for _ in range(nreq):
        grp = 0 if (with_group and rng.random() < 0.6) else -1
        lo = gp[0] * 16 + 1 if grp == 0 else 1
        ctx = int(rng.integers(max(lo, 1), 301))
        ctx = max(ctx, lo)
        ql_max = min(70, ctx - (gp[0] * 16 if grp == 0 else 0))
        ql = int(rng.integers(1, ql_max + 1))
        reqs.append(W.ReqSpec(W.OFFLINE_PREFILL if ql > 1 else W.ONLINE_DECODE, ctx, ql, grp))
    return W.custom_config("rand", Hkv * g, Hkv, d, seed, reqs, gp)


@pytest.mark.parametrize("d,g,seed", [(64, 1, 0), (128, 4, 1), (64, 5, 2), (128, 8, 3),
                                      (64, 1, 4), (128, 1, 5)])
def test_dense_numpy(d, g, seed):
    rng = np.random.default_rng(seed)
    cfg = _random_cfg(rng, d, g, seed=seed, with_group=bool(seed % 2))
    wl = W.make_workload(cfg, preappended=True)
    b, kp, vp, q = _post_state(wl)
    st, out, lse = oracle.attention(b, kp, vp, q)
    assert st == oracle.OK
    ref, ref_lse = _dense_reference(b, kp, vp, q)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(lse, ref_lse, rtol=0, atol=1e-12)


def test_torch_sdpa_fp64():
    rng = np.random.default_rng(11)
    cfg = _random_cfg(rng, 64, 4, Hkv=2, nreq=4, seed=11)
    wl = W.make_workload(cfg, preappended=True)
    b, kp, vp, q = _post_state(wl)
    st, out, _ = oracle.attention(b, kp, vp, q)
    assert st == oracle.OK
    Hq, Hkv = b["num_q_heads"], b["num_kv_heads"]
    for i in range(b["num_reqs"]):
        q0, q1 = b["q_indptr"][i], b["q_indptr"][i + 1]
        ql, ctx = q1 - q0, int(b["ctx_len"][i])
        K = torch.stack([torch.from_numpy(_gather_dense(b, _bf16_to_f64(kp), i, h))
                         for h in range(Hkv)])
        V = torch.stack([torch.from_numpy(_gather_dense(b, _bf16_to_f64(vp), i, h))
                         for h in range(Hkv)])
        Q = torch.from_numpy(_bf16_to_f64(q)[q0:q1]).permute(1, 0, 2)  # [Hq][ql][d]
        mask = torch.arange(ctx)[None, :] <= torch.arange(ctx - ql, ctx)[:, None]
        ref = torch.nn.functional.scaled_dot_product_attention(
            Q[None], K[None], V[None], attn_mask=mask, enable_gqa=True)[0]
        np.testing.assert_allclose(out[q0:q1], ref.permute(1, 0, 2).numpy(), atol=1e-12, rtol=0)


def test_ctx1_closed_form():
    cfg = W.custom_config("c1", 2, 2, 64, 5, [W.ReqSpec(W.ONLINE_DECODE, 1, 1)], [])
    wl = W.make_workload(cfg, preappended=True)
    b, kp, vp, q = _post_state(wl)
    st, out, lse = oracle.attention(b, kp, vp, q)
    assert st == oracle.OK
    blk = b["block_table"][0, 0]
    for h in range(2):
        v0 = _bf16_to_f64(vp)[blk, h, 0]
        k0 = _bf16_to_f64(kp)[blk, h, 0]
        assert np.array_equal(out[0, h], v0)  # exact: w=1, Z=1
        expect = float(np.dot(_bf16_to_f64(q)[0, h], k0)) / 8.0
        assert abs(lse[0, h] - expect) <= 1e-12 * max(1.0, abs(expect))


def test_constant_v():
    cfg = W.custom_config("cv", 4, 2, 64, 6, [W.ReqSpec(W.OFFLINE_PREFILL, 77, 20),
                                             W.ReqSpec(W.ONLINE_DECODE, 130, 1)], [])
    wl = W.make_workload(cfg, preappended=True)
    c = torch.linspace(-2, 2, 64).to(torch.bfloat16)
    vp = wl.v_pool.clone()
    vp[:] = c
    st, out, _ = oracle.attention(wl.batch, wl.k_pool, vp, wl.q)
    assert st == oracle.OK
    assert np.max(np.abs(out - c.double().numpy())) <= 1e-14  # ~n*eps*|c| rounding of the weighted sum


def test_equal_keys_cumulative_mean():
    """All K rows equal -> row p: O = mean(v_0..v_p), lse = s q.k + ln(p+1)."""
    cfg = W.custom_config("ek", 2, 1, 64, 7, [W.ReqSpec(W.OFFLINE_PREFILL, 50, 50)], [])
    wl = W.make_workload(cfg, preappended=True)
    kp = wl.k_pool.clone()
    k = torch.randn(64).to(torch.bfloat16)
    kp[:] = k
    b = wl.batch
    st, out, lse = oracle.attention(b, kp, wl.v_pool, wl.q)
    assert st == oracle.OK
    V = _gather_dense(b, _bf16_to_f64(wl.v_pool), 0, 0)
    kd = k.double().numpy()
    for p in range(50):
        for h in range(2):
            np.testing.assert_allclose(out[p, h], V[: p + 1].mean(axis=0), atol=1e-12, rtol=0)
            e = float(_bf16_to_f64(wl.q)[p, h] @ kd) / 8.0 + math.log(p + 1)
            assert abs(lse[p, h] - e) <= 1e-12 * max(1, abs(e))


def test_spike_limit():
    """q = 50 k_j/|k_j| -> O -> v_j."""
    cfg = W.custom_config("sp", 1, 1, 64, 8, [W.ReqSpec(W.ONLINE_DECODE, 40, 1)], [])
    wl = W.make_workload(cfg, preappended=True)
    b = wl.batch
    K = _gather_dense(b, _bf16_to_f64(wl.k_pool), 0, 0)
    V = _gather_dense(b, _bf16_to_f64(wl.v_pool), 0, 0)
    j = 17
    qv = 50.0 * K[j] / np.linalg.norm(K[j])
    q = torch.from_numpy(qv).to(torch.bfloat16).reshape(1, 1, 64)
    st, out, _ = oracle.attention(b, wl.k_pool, wl.v_pool, q)
    assert st == oracle.OK
    np.testing.assert_allclose(out[0, 0], V[j], atol=1e-6, rtol=0)


def test_block_permutation_invariance():
    rng = np.random.default_rng(21)
    cfg = _random_cfg(rng, 64, 2, seed=21, with_group=True)
    wl = W.make_workload(cfg, preappended=True)
    b = wl.batch
    st, out, lse = oracle.attention(b, wl.k_pool, wl.v_pool, wl.q)
    perm = torch.randperm(b["num_blocks"], generator=torch.Generator().manual_seed(5))
    kp2 = torch.empty_like(wl.k_pool)
    vp2 = torch.empty_like(wl.v_pool)
    kp2[perm] = wl.k_pool
    vp2[perm] = wl.v_pool
    b2 = dict(b)
    bt = b["block_table"].copy()
    bt[bt >= 0] = perm.numpy()[bt[bt >= 0]]
    b2["block_table"] = bt
    st2, out2, lse2 = oracle.attention(b2, kp2, vp2, wl.q)
    assert st == st2 == oracle.OK
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_shared_equals_duplicated_prefix():
    """Reading #7: sharing storage does not change the result (bit-exact in the oracle)."""
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 100, 30, 0), W.ReqSpec(W.OFFLINE_DECODE, 90, 1, 0)]
    cfg = W.custom_config("sh", 4, 2, 64, 9, reqs, [3])
    wl = W.make_workload(cfg, preappended=True)
    b = wl.batch
    st, out, lse = oracle.attention(b, wl.k_pool, wl.v_pool, wl.q)
    assert st == oracle.OK
    # physically duplicate the prefix for request 1 into fresh blocks
    n0 = b["num_blocks"]
    kp = torch.cat([wl.k_pool, wl.k_pool[b["block_table"][1, :3]]])
    vp = torch.cat([wl.v_pool, wl.v_pool[b["block_table"][1, :3]]])
    b2 = dict(b)
    bt = b["block_table"].copy()
    bt[1, :3] = np.arange(n0, n0 + 3)
    b2["block_table"] = bt
    b2["group_of"] = np.array([-1, -1], np.int32)
    b2["group_prefix_blocks"] = np.zeros(0, np.int32)
    b2["num_blocks"] = n0 + 3
    st2, out2, lse2 = oracle.attention(b2, kp, vp, wl.q)
    assert st2 == oracle.OK
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_chunking_and_decode_vs_prefill():
    """A prompt done as one chunk == n chunks; a decode at p == row p of the prefill."""
    full = W.custom_config("cf", 4, 2, 64, 10, [W.ReqSpec(W.OFFLINE_PREFILL, 120, 120)], [])
    wl = W.make_workload(full, preappended=True)
    b = wl.batch
    st, out, lse = oracle.attention(b, wl.k_pool, wl.v_pool, wl.q)
    assert st == oracle.OK
    for lo, hi in [(0, 37), (37, 80), (80, 119), (119, 120)]:
        bc = dict(b)
        bc["q_indptr"] = np.array([0, hi - lo], np.int32)
        bc["ctx_len"] = np.array([hi], np.int32)
        st2, o2, l2 = oracle.attention(bc, wl.k_pool, wl.v_pool, wl.q[lo:hi])
        assert st2 == oracle.OK
        np.testing.assert_allclose(o2, out[lo:hi], atol=1e-12, rtol=0)
        np.testing.assert_allclose(l2, lse[lo:hi], atol=1e-12, rtol=0)


def test_gqa_equals_repeated_mha():
    rng = np.random.default_rng(31)
    cfg = _random_cfg(rng, 64, 4, Hkv=2, seed=31)
    wl = W.make_workload(cfg, preappended=True)
    b = wl.batch
    st, out, lse = oracle.attention(b, wl.k_pool, wl.v_pool, wl.q)
    assert st == oracle.OK
    b2 = dict(b)
    b2["num_kv_heads"] = b["num_q_heads"]
    kp = wl.k_pool.repeat_interleave(4, dim=1)
    vp = wl.v_pool.repeat_interleave(4, dim=1)
    st2, out2, lse2 = oracle.attention(b2, kp, vp, wl.q)
    assert st2 == oracle.OK
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_lse_merge_identity():
    """Oracle over A u B == LSE-merge of dense partials over A and B (the a6 closed form)."""
    cfg = W.custom_config("mg", 2, 1, 64, 12, [W.ReqSpec(W.ONLINE_DECODE, 200, 1)], [])
    wl = W.make_workload(cfg, preappended=True)
    b = wl.batch
    st, out, lse = oracle.attention(b, wl.k_pool, wl.v_pool, wl.q)
    K = _gather_dense(b, _bf16_to_f64(wl.k_pool), 0, 0)
    V = _gather_dense(b, _bf16_to_f64(wl.v_pool), 0, 0)
    qd = _bf16_to_f64(wl.q)[0]
    for h in range(2):
        parts = []
        for lo, hi in [(0, 64), (64, 200)]:
            x = K[lo:hi] @ qd[h] / 8.0
            m = x.max()
            w = np.exp(x - m)
            parts.append(((w @ V[lo:hi]) / w.sum(), m + np.log(w.sum())))
        L = np.logaddexp(parts[0][1], parts[1][1])
        O = sum(np.exp(l - L) * o for o, l in parts)
        np.testing.assert_allclose(O, out[0, h], atol=1e-12, rtol=0)
        assert abs(L - lse[0, h]) < 1e-12


def test_validation_errors():
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 100, 30, 0), W.ReqSpec(W.OFFLINE_DECODE, 90, 1, 0)]
    cfg = W.custom_config("v", 4, 2, 64, 13, reqs, [3])
    wl = W.make_workload(cfg, preappended=True)
    b = dict(wl.batch)
    assert oracle.validate(b) == oracle.OK
    bad = dict(b)
    bad["group_prefix_blocks"] = np.array([7], np.int32)  # 112 > 90-1: queries inside prefix
    assert oracle.validate(bad) == oracle.GROUP
    bad = dict(b)
    bt = b["block_table"].copy()
    bt[1, 0] = bt[1, 5]  # member's first block differs from the group's
    bad["block_table"] = bt
    assert oracle.validate(bad) == oracle.GROUP
    bad = dict(b)
    bad["q_indptr"] = np.array([0, 101, 102], np.int32)  # q_len > ctx
    assert oracle.validate(bad) == oracle.INVALID
    bad = dict(b)
    bad["num_q_heads"] = 3  # Hq % Hkv != 0
    assert oracle.validate(bad) == oracle.INVALID


@pytest.mark.parametrize("d,g,seed", [(64, 1, 21), (128, 4, 22), (64, 5, 23)])
def test_attention_rows_pinned(d, g, seed):
    """orc_attention_rows (the reference of every full-size sampled GPU test and of the
    cpu_baseline) against the dense numpy textbook definition, row by row, and bit-exactly
    against orc_attention: every request's first and last query row (request boundaries,
    including its causal diagonal) plus random rows, every head, in shuffled order."""
    rng = np.random.default_rng(seed)
    cfg = _random_cfg(rng, d, g, nreq=5, seed=seed, with_group=True)
    wl = W.make_workload(cfg, preappended=True)
    b, kp, vp, q = _post_state(wl)
    qi = np.asarray(b["q_indptr"])
    Hq = b["num_q_heads"]
    bnd = sorted({int(x) for i in range(b["num_reqs"]) for x in (qi[i], qi[i + 1] - 1)})
    rnd = rng.integers(0, int(qi[-1]), 40).tolist()
    rows = np.array([r for r in bnd + rnd for _ in range(Hq)], np.int32)
    heads = np.array([h for _ in bnd + rnd for h in range(Hq)], np.int32)
    perm = rng.permutation(len(rows))
    rows, heads = rows[perm], heads[perm]
    st, o_rows, l_rows = oracle.attention_rows(b, kp, vp, q, rows, heads, nthreads=3)
    assert st == oracle.OK
    ref, ref_lse = _dense_reference(b, kp, vp, q)
    np.testing.assert_allclose(o_rows, ref[rows, heads], rtol=0, atol=1e-12)
    np.testing.assert_allclose(l_rows, ref_lse[rows, heads], rtol=0, atol=1e-12)
    st, full, full_lse = oracle.attention(b, kp, vp, q)
    assert np.array_equal(o_rows, full[rows, heads]) and np.array_equal(l_rows, full_lse[rows, heads])
    # out-of-range rows / heads are rejected
    assert oracle.attention_rows(b, kp, vp, q, [int(qi[-1])], [0])[0] == oracle.INVALID
    assert oracle.attention_rows(b, kp, vp, q, [0], [Hq])[0] == oracle.INVALID
