"""GPU parity of the launch modes selected by kva_set_option (include/kvattn.h): the tile kernel
overlapped with decode (programmatic dependent launch on one stream, or two streams) vs run
after it, forced tile-kernel grid sizes, and the cooperative evict_select grid size — each
against the oracle and, where the arithmetic is the same, bit-exactly against each other."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W
from gpu_util import assert_attention_close, gpu_step, oracle_step

pytestmark = pytest.mark.gpu


def _mixed(d, Hq, Hkv):
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 600 + 300, 300, 0), W.ReqSpec(W.OFFLINE_PREFILL, 600 + 173, 173, 0),
            W.ReqSpec(W.ONLINE_DECODE, 2000, 1), W.ReqSpec(W.ONLINE_DECODE, 77, 1)]
    reqs += [W.ReqSpec(W.OFFLINE_DECODE, 600 + 5 + i, 1, 0) for i in range(20)]
    reqs += [W.ReqSpec(W.OFFLINE_DECODE, 1100, 2), W.ReqSpec(W.OFFLINE_DECODE, 730, 2, 0)]
    return W.make_workload(W.custom_config("v", Hq, Hkv, d, 7, reqs, [600 // 16]))


MODES = {"pdl": dict(overlap=1, pdl=1), "pdl_fold": dict(overlap=1, pdl=1, fold=1), "two_streams": dict(overlap=1, pdl=0),
         "sequential": dict(overlap=0), "tile40": dict(overlap=1, tile_ctas=40),
         "tile1": dict(overlap=1, tile_ctas=1)}


@pytest.mark.parametrize("d,Hq,Hkv", [(128, 16, 2), (64, 8, 4)])
def test_launch_modes_match_oracle_and_each_other(d, Hq, Hkv):
    import paper_2504_03651_b200 as K
    wl = _mixed(d, Hq, Hkv)
    r = oracle_step(wl)
    outs = {}
    for name, opts in MODES.items():
        with K.options(**opts):
            g = gpu_step(wl)
        assert_attention_close(g["out"], g["lse"], r["out"], r["lse"])
        outs[name] = g["out"].cpu().numpy()
    # the same tile items and splits in every mode: the arithmetic does not depend on the schedule
    for name, o in outs.items():
        assert np.array_equal(o, outs["pdl"]), name


def test_pdl_merge_waits_for_the_tile_kernel():
    """Under PDL the decode kernel may start (and finish) while the tile kernel still runs; the
    merge after it reads cascade partials the TILE kernel writes.  Force the tile kernel to be
    the long pole (1 persistent CTA, a long prefill chunk in the batch) with the workspace
    NaN-filled: a merge that did not wait for it would produce NaN / wrong rows."""
    import paper_2504_03651_b200 as K
    reqs = [W.ReqSpec(W.OFFLINE_DECODE, 40 * 16 + 3 + i, 1, 0) for i in range(12)]
    reqs += [W.ReqSpec(W.OFFLINE_PREFILL, 40 * 16 + 1500, 1500, 0), W.ReqSpec(W.ONLINE_DECODE, 900, 1)]
    wl = W.make_workload(W.custom_config("pdl", 16, 2, 128, 61, reqs, [40]))
    dev = "cuda"
    with K.options(tile_ctas=1, overlap=1, pdl=1):
        pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), K.free_bits_tensor(wl.free_bits, dev))
        batch = K.Batch(wl.batch, dev)
        K.kv_append(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
        ws = torch.full((K.hybrid_attention_workspace_size(batch) // 4 + 64,), float("nan"),
                        device=dev).view(torch.uint8)
        plan = K.Plan(pool, batch, ws)
        assert plan.stats()["n_cascade_items"] > 0
        q = wl.q.to(dev)
        out = torch.empty(q.shape, dtype=torch.float32, device=dev)
        lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
        plan.run(q, out, lse)
        torch.cuda.synchronize()
    r = oracle_step(wl)
    assert_attention_close(out, lse, r["out"], r["lse"])


@pytest.mark.parametrize("ctas", [1, 7, 148, 296])
def test_evict_select_grid_sizes(ctas):
    """The selection's per-CTA bin reservations and segment ranges give the oracle's eviction
    order for any cooperative grid size (option evict_ctas), on the full-size `evict` config, its
    straddle variant and a skewed adversarial case."""
    import paper_2504_03651_b200 as K
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()  # noqa: E731
    with K.options(evict_ctas=ctas):
        for straddle in (False, True):
            ev = W.make_evict(straddle=straddle)
            keys = K.evict_keys(t(ev.state, np.uint8), t(ev.rc, np.int32), t(ev.lat, np.int32),
                                t(ev.depth, np.int16))
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


def test_truncate_after_a_run_without_merge_waits_for_the_tile_kernel():
    """A run whose last kernel is the decode kernel (every decode direct: no split, no group, so
    no merge) with the tile kernel as the long pole (1 persistent CTA): kv_truncate right after
    it resets the chunk's new table entries, and its release kernel is a programmatic dependent
    that waits only for its predecessor — the join kernel that ends such a run must make that
    the tile kernel as well, else the tile kernel reads -1 entries (zero-filled K/V)."""
    import paper_2504_03651_b200 as K
    reqs = [W.ReqSpec(W.OFFLINE_PREFILL, 2400, 2000, -1), W.ReqSpec(W.ONLINE_DECODE, 300, 1),
            W.ReqSpec(W.ONLINE_DECODE, 500, 1)]
    wl = W.make_workload(W.custom_config("join", 16, 2, 128, 67, reqs, []))
    dev = "cuda"
    r = oracle_step(wl)
    for _ in range(3):
        with K.options(tile_ctas=1, overlap=1, pdl=1):
            pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), K.free_bits_tensor(wl.free_bits, dev))
            batch = K.Batch(wl.batch, dev)
            plan = K.kv_append_plan(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
            st = plan.stats()
            assert st["n_merge_rows"] == 0 and st["n_tile_items"] > 0 and st["n_decode_items"] > 0
            assert plan.launch_count() == 3  # tile, decode, join
            q = wl.q.to(dev)
            out = torch.empty(q.shape, dtype=torch.float32, device=dev)
            lse = torch.empty(q.shape[:2], dtype=torch.float32, device=dev)
            plan.run(q, out, lse)
            keep = (wl.batch["ctx_len"] - np.diff(wl.batch["q_indptr"])).astype(np.int32)
            K.kv_truncate(pool, batch, keep)
            torch.cuda.synchronize()
        assert_attention_close(out, lse, r["out"], r["lse"])


def test_fold_merges_members_in_the_decode_epilogue():
    """Option fold: the decode-class members of a one-level group whose suffix is one split
    merge their suffix partial with the cascade partial in the decode kernel's epilogue (waiting
    on the tile kernel's per-item completion counters); the merge kernel gets the remaining
    requests.  Results equal the merge-kernel path bit-exactly and the oracle within
    tolerance, across repeated runs of one plan (the counters' epochs) and a tile kernel on one
    CTA (the decode warps wait for it)."""
    import paper_2504_03651_b200 as K
    wl = _mixed(128, 16, 2)
    r = oracle_step(wl)
    dev = "cuda"
    outs = []
    for opts in (dict(fold=0), dict(fold=1), dict(fold=1, tile_ctas=1)):
        with K.options(overlap=1, pdl=1, **opts):
            pool = K.Pool(wl.k_pool.to(dev), wl.v_pool.to(dev), K.free_bits_tensor(wl.free_bits, dev))
            batch = K.Batch(wl.batch, dev)
            plan = K.kv_append_plan(pool, batch, wl.k_new.to(dev), wl.v_new.to(dev))
            q = wl.q.to(dev)
            for _ in range(3):
                out = torch.full(q.shape, float("nan"), dtype=torch.float32, device=dev)
                lse = torch.full(q.shape[:2], float("nan"), dtype=torch.float32, device=dev)
                plan.run(q, out, lse)
                torch.cuda.synchronize()
                assert_attention_close(out, lse, r["out"], r["lse"])
                outs.append((out.cpu().numpy(), lse.cpu().numpy()))
    for o, l in outs[1:]:
        assert np.array_equal(o, outs[0][0]) and np.array_equal(l, outs[0][1])
