"""GPU parity for evict_keys / evict_select: bit-exact keys and eviction order vs the oracle
(S:146)."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a).view(dtype)).cuda()


def _gpu_keys(ev):
    import paper_2504_03651_b200 as K
    st = _dev(ev.state, np.uint8)
    rc = _dev(ev.rc.view(np.int32), np.int32)
    lat = _dev(ev.lat.view(np.int32), np.int32)
    dep = _dev(ev.depth.view(np.int16), np.int16) if ev.depth is not None else None
    return K.evict_keys(st, rc, lat, dep)


@pytest.mark.parametrize("straddle", [False, True])
def test_evict_full_size(straddle):
    import paper_2504_03651_b200 as K
    ev = W.make_evict(straddle=straddle)
    keys = _gpu_keys(ev)
    s, ref_keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    torch.cuda.synchronize()
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), ref_keys)
    ids, n = K.evict_select(keys, ev.k)
    s, ref_ids = oracle.evict_select(ref_keys, ev.k)
    assert n == len(ref_ids) == ev.k
    assert np.array_equal(ids.cpu().numpy(), ref_ids)


@pytest.mark.parametrize("seed", range(6))
def test_evict_random_small(seed):
    import paper_2504_03651_b200 as K
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 50000))
    ev = W.make_evict(n=n, k=int(rng.integers(1, n + 10)), seed=seed, run_lo=1, run_hi=9)
    # force many equal keys: coarse lat
    ev.lat[:] = ev.lat % 3
    keys = _gpu_keys(ev)
    s, ref_keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    ids, nsel = K.evict_select(keys, ev.k)
    s2, ref_ids = oracle.evict_select(ref_keys, ev.k)
    assert nsel == len(ref_ids)
    assert np.array_equal(ids.cpu().numpy(), ref_ids)


@pytest.mark.parametrize("n,k", [(4096, 100), (1 << 20, 1 << 16)])
def test_evict_apply_marks_free(n, k):
    """apply = 1: the device free bitmap and the pool's host mirror
    afterwards equal the oracle's evict_select_apply on the same pre-existing bitmap (the
    state-0 blocks free), bit-exact, at a small size and at the full `evict` size."""
    import paper_2504_03651_b200 as K
    ev = W.make_evict(n=n, k=k, seed=9)
    keys = _gpu_keys(ev)
    bits = np.zeros((n + 31) // 32, np.uint32)
    idx = np.nonzero(ev.state == 0)[0]
    np.bitwise_or.at(bits, idx // 32, np.uint32(1) << (idx % 32).astype(np.uint32))
    _, ref_keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    s, ref_ids, ref_bits = oracle.evict_select_apply(ref_keys, k, bits)
    kp = torch.zeros((n, 1, 16, 64), dtype=torch.bfloat16, device="cuda")
    fb = K.free_bits_tensor(bits, "cuda")
    pool = K.Pool(kp, kp, fb)
    n0 = pool.free_count()
    ids, nsel = K.evict_select(keys, k, apply=True, pool=pool)
    torch.cuda.synchronize()
    assert nsel == len(ref_ids) and np.array_equal(ids.cpu().numpy(), ref_ids)
    assert np.array_equal(fb.cpu().numpy().view(np.uint32), ref_bits)
    assert pool.free_count() == n0 + nsel
    pool.resync()                       # the mirror re-read from the device agrees
    assert pool.free_count() == n0 + nsel


def test_evict_short():
    import paper_2504_03651_b200 as K
    st = np.array([1, 2, 5, 4, 0], np.uint8)
    ev = W.EvictWorkload(st, np.zeros(5, np.uint32), np.arange(5, dtype=np.uint32),
                         np.zeros(5, np.uint16), 4, None, None)
    keys = _gpu_keys(ev)
    ids, n = K.evict_select(keys, 4)
    assert n == 2 and list(ids.cpu().numpy()) == [2, 3]


def test_release_blocks_roundtrip_and_errors():
    """kv_release_blocks returns blocks to the pool (P:448 recompute-mode release); a second
    kv_append then re-allocates exactly those ids (smallest free first, reading #13)."""
    import paper_2504_03651_b200 as K
    wl = W.make_workload("tiny")
    dev = "cuda"
    fb = K.free_bits_tensor(wl.free_bits, dev)
    pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), fb)
    batch = K.Batch(wl.batch, dev)
    n0 = pool.free_count()
    pristine = wl.batch["block_table"]
    K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
    new_ids = batch.table_host[(pristine == -1) & (batch.table_host >= 0)]
    assert pool.free_count() == n0 - len(new_ids)
    with pytest.raises(K.KvaError):            # double release of a free block
        K.kv_release_blocks(pool, np.array([int(np.nonzero(np.unpackbits(
            wl.free_bits.view(np.uint8), bitorder="little"))[0][-1])], np.int32))
    with pytest.raises(K.KvaError):            # listed twice
        K.kv_release_blocks(pool, np.array([new_ids[0], new_ids[0]], np.int32))
    fb_before = fb.cpu().numpy().view(np.uint32).copy()
    s_ref, fb_ref = oracle.release_blocks(fb_before, wl.batch["num_blocks"], new_ids)
    assert s_ref == oracle.OK
    K.kv_release_blocks(pool, new_ids)
    torch.cuda.synchronize()
    assert np.array_equal(fb.cpu().numpy().view(np.uint32), fb_ref)
    assert pool.free_count() == n0
    assert np.array_equal(fb.cpu().numpy().view(np.uint32), wl.free_bits)
    batch2 = K.Batch(wl.batch, dev)
    K.kv_append(pool, batch2, wl.k_new.to(dev), wl.v_new.to(dev))
    assert np.array_equal(batch2.table_host, batch.table_host)


def test_evict_k_larger_than_evictable_and_zero():
    import paper_2504_03651_b200 as K
    ev = W.make_evict(n=3000, k=10, seed=11)
    keys = _gpu_keys(ev)
    s, ref_keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    n_ev = int((ref_keys != np.uint64(0xFFFFFFFFFFFFFFFF)).sum())
    ids, n = K.evict_select(keys, n_ev + 100)
    s2, ref_ids = oracle.evict_select(ref_keys, n_ev + 100)
    assert n == n_ev and np.array_equal(ids.cpu().numpy(), ref_ids)
    ids, n = K.evict_select(keys, 0)
    assert n == 0


_ADV = ["all_equal", "two_values", "short", "k1", "k_all", "clustered", "few_ev", "outliers_half",
        "take_all_skewed", "many_runs", "fin_bucket", "deep_ties"]


def _adversarial(case, n):
    rng = np.random.default_rng(sum(map(ord, case)))
    keys = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    k = 5000
    if case == "all_equal":
        keys[:] = np.uint64(12345)
    elif case == "two_values":
        keys = np.where(rng.random(n) < 0.5, np.uint64(7), np.uint64(9)).astype(np.uint64)
    elif case == "short":
        keys[rng.random(n) < 0.97] = np.uint64(0xFFFFFFFFFFFFFFFF)
        k = 10000
    elif case == "k1":
        k = 1
    elif case == "k_all":
        k = n
    elif case == "clustered":
        keys = (np.uint64(1 << 40) + rng.integers(0, 3000, n).astype(np.uint64)).astype(np.uint64)
    elif case == "few_ev":
        keys[:] = np.uint64(0xFFFFFFFFFFFFFFFF)
        keys[rng.choice(n, 37, replace=False)] = rng.integers(0, 100, 37).astype(np.uint64)
        k = 20
    elif case == "outliers_half":
        # almost every key equal, a few outliers far above: the k-th key's bin holds nearly all
        # keys round after round (segment rounds down to the id bits)
        keys[:] = np.uint64(5)
        idx = rng.choice(n, 64, replace=False)
        keys[idx] = (np.uint64(1) << np.uint64(60)) + rng.integers(0, 1 << 40, 64).astype(np.uint64)
        k = n // 2
    elif case == "take_all_skewed":
        # E <= k and one taken bin far larger than a CTA sort: partitioned bucket levels
        keys[:] = np.uint64(1)
        idx = rng.choice(n, n // 10, replace=False)
        keys[idx] = rng.integers(1 << 50, 1 << 61, len(idx)).astype(np.uint64)
        k = n + 7
    elif case == "many_runs":
        # varying bits in 32 separate runs (more than the kernel keeps apart: gaps merged)
        keys = (rng.integers(0, 1 << 63, n, dtype=np.uint64) & np.uint64(0x5555555555555555)).astype(np.uint64)
        k = 3 * n // 4
    elif case == "fin_bucket":
        # the k-th key's bin is small: finished by one sort with take < size
        keys = rng.integers(0, 1 << 20, n, dtype=np.uint64)
        k = 777
    elif case == "deep_ties":
        # 3 distinct keys; k inside the middle one, ties broken by id deep in the id bits
        keys = rng.choice(np.array([3, 1 << 33, (1 << 33) + 1], np.uint64), n).astype(np.uint64)
        k = n // 2 + 3
    return keys, k


@pytest.mark.parametrize("case", _ADV)
def test_select_adversarial(case):
    """n = 2^17: heavy ties, fewer evictable blocks than k, k = 1, k = n, clustered keys, very
    few evictable blocks, a boundary bin that stays huge for several rounds, taken bins larger
    than a CTA sort (partition levels), > 8 runs of varying bits, a finish-sorted boundary bin."""
    import paper_2504_03651_b200 as K
    n = 1 << 17
    keys, k = _adversarial(case, n)
    d = torch.from_numpy(keys.view(np.int64)).cuda()
    ids, nsel = K.evict_select(d, k)
    s, ref = oracle.evict_select(keys, k)
    assert nsel == len(ref)
    assert np.array_equal(ids.cpu().numpy(), ref)


@pytest.mark.parametrize("n", [1, 2, 3, 31, 1000, 4099, 65537])
def test_select_small_odd_and_unaligned(n):
    """Odd n (the last slice's odd tail) and a keys pointer that is not 16-B aligned (scalar loads)."""
    import paper_2504_03651_b200 as K
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << 12, n + 1, dtype=np.uint64)
    keys[rng.random(n + 1) < 0.1] = np.uint64(0xFFFFFFFFFFFFFFFF)
    d = torch.from_numpy(keys.view(np.int64)).cuda()
    for off in (0, 1):
        kk = keys[off:off + n]
        for k in {1, max(1, n // 3), n}:
            ids, nsel = K.evict_select(d[off:off + n], k)
            s, ref = oracle.evict_select(kk, k)
            assert nsel == len(ref)
            assert np.array_equal(ids.cpu().numpy(), ref), (off, k)


@pytest.mark.parametrize("cfg", ["tiny", "qwen14b"])
def test_truncate_rollback_matches_oracle(cfg):
    """kv_truncate: after kv_append, truncating every request to its pre-append length
    gives the oracle's table (host mirror AND device table) and free bitmap — the pristine
    ones — and the next kv_append re-allocates exactly the same ids (smallest free first)."""
    import paper_2504_03651_b200 as K
    wl = W.make_workload(cfg)
    dev = "cuda"
    fb = K.free_bits_tensor(wl.free_bits, dev)
    pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), fb)
    batch = K.Batch(wl.batch, dev)
    n0 = pool.free_count()
    K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
    after = batch.table_host.copy()
    keep = (wl.batch["ctx_len"] - np.diff(wl.batch["q_indptr"])).astype(np.int32)
    s, fb_ref, bt_ref = oracle.truncate(dict(wl.batch, block_table=after), fb.cpu().numpy().view(np.uint32), keep)
    assert s == oracle.OK
    K.kv_truncate(pool, batch, keep)
    torch.cuda.synchronize()
    assert np.array_equal(batch.table_host, bt_ref) and np.array_equal(bt_ref, wl.batch["block_table"])
    assert np.array_equal(batch.table_dev.cpu().numpy(), bt_ref)
    assert np.array_equal(fb.cpu().numpy().view(np.uint32), fb_ref)
    assert pool.free_count() == n0
    K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
    assert np.array_equal(batch.table_host, after)
    with pytest.raises(K.KvaError):  # keep > ctx
        K.kv_truncate(pool, batch, wl.batch["ctx_len"] + 1)


@pytest.mark.parametrize("case", _ADV + ["evict", "straddle"])
def test_select_256_thread_build(case):
    """The 256-thread build (option evict_threads = 256: 1,024-pair CTA buckets, 7-bit warp
    digits, the warp areas inside the round buffer) gives the oracle's order bit-exactly on the
    adversarial cases and the full-size `evict` config (+ straddle)."""
    import paper_2504_03651_b200 as K
    if case in ("evict", "straddle"):
        ev = W.make_evict(straddle=case == "straddle")
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()  # noqa: E731
        d = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32), t(ev.depth, np.int16))
        keys = d.cpu().numpy().view(np.uint64)
        k = ev.k
    else:
        keys, k = _adversarial(case, 1 << 17)
        d = torch.from_numpy(keys.view(np.int64)).cuda()
    s, ref = oracle.evict_select(keys, k)
    for ctas in (0, 37):
        with K.options(evict_threads=256, evict_ctas=ctas):
            ids, nsel = K.evict_select(d, k)
        assert nsel == len(ref)
        assert np.array_equal(ids.cpu().numpy(), ref), ctas
    with pytest.raises(K.KvaError):
        K.set_option("evict_threads", 300)
