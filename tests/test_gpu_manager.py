"""GPU parity of the KV-manager step and the burst-reserve threshold of
kv_append, through the C ABI, against the oracle (bit-exact: state, rc, lat, keys, active
count, eviction order, block tables)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2504_03651_b200 as K
import workloads as W

pytestmark = pytest.mark.gpu


def _dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("seed", range(8))
def test_manager_random_sequences(seed):
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(50, 3000))
    state = rng.integers(0, 6, n).astype(np.uint8)
    lat = rng.integers(0, 100, n).astype(np.uint32)
    depth = rng.integers(0, 8, n).astype(np.uint16)
    rc = np.zeros(n, np.uint32)
    d_state, d_lat, d_rc = _dev(state, np.uint8), _dev(lat, np.int32), _dev(rc, np.int32)
    d_depth = _dev(depth, np.int16)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, d_depth)
    for it in range(4):
        now = 1000 + it
        # overlapping chains on purpose: the last chain wins (list order)
        chains = [(int(rng.integers(0, 6)), rng.choice(n, int(rng.integers(1, 40)), replace=False))
                  for _ in range(int(rng.integers(0, 12)))]
        pool = [rng.choice(n, int(rng.integers(1, 60)), replace=False) for _ in range(int(rng.integers(0, 30)))]
        pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda() if pool else None
        keys = mgr(now, chains, pool_ids)
        torch.cuda.synchronize()
        st, state, rc, lat, rkeys, nact = oracle.manager_step(state, rc, lat, depth, now, chains, pool)
        assert st == oracle.OK
        assert np.array_equal(d_state.cpu().numpy(), state)
        assert np.array_equal(_u32(d_rc), rc)
        assert np.array_equal(_u32(d_lat), lat)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
        assert int(mgr.n_active.item()) == nact
        k = int(rng.integers(1, n))
        ids, nsel = K.evict_select(keys, k)
        _, rids = oracle.evict_select(rkeys, k)
        assert np.array_equal(ids.cpu().numpy(), rids)


def test_manager_full_size_evict_config():
    """The `evict` config (2^20 blocks, 90% resident): an offline pool whose chains reproduce the
    drawn rc (126k pool requests, 9.1M block references), 5% of runs touched, 1% finishing;
    then the top-64k selection."""
    ev = W.make_evict()
    chains, pool = W.make_manager_update(ev, now=1 << 20, seed=1)
    rc0 = np.zeros(len(ev.state), np.uint32)
    d_state, d_lat = _dev(ev.state, np.uint8), _dev(ev.lat, np.int32)
    d_rc, d_depth = _dev(rc0, np.int32), _dev(ev.depth, np.int16)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, d_depth)
    pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda()
    keys = mgr(1 << 20, chains, pool_ids)
    ids, nsel = K.evict_select(keys, ev.k)
    st, state, rc, lat, rkeys, nact = oracle.manager_step(ev.state, rc0, ev.lat, ev.depth, 1 << 20, chains, pool)
    assert st == oracle.OK
    assert np.array_equal(_u32(d_rc), rc)
    assert np.array_equal(rc[ev.state == W.EV_ACTIVE_OFFLINE], ev.rc[ev.state == W.EV_ACTIVE_OFFLINE])
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
    assert int(mgr.n_active.item()) == nact
    _, rids = oracle.evict_select(rkeys, ev.k)
    assert np.array_equal(ids.cpu().numpy(), rids)


def test_manager_incremental_counts():
    """Incremental mode: the `evict` config's pool, 1% of its requests leave and new ones join;
    rc / keys / eviction order equal the oracle's (which equals a full recount of the new pool,
    tests/test_oracle_manager.py)."""
    ev = W.make_evict()
    chains, pool = W.make_manager_update(ev, now=1 << 20, seed=2)
    rng = np.random.default_rng(9)
    leave = [pool[i] for i in rng.choice(len(pool), len(pool) // 100, replace=False)]
    join = [pool[i] for i in rng.choice(len(pool), len(pool) // 100, replace=False)]
    d_state, d_lat = _dev(ev.state, np.uint8), _dev(ev.lat, np.int32)
    d_rc, d_depth = _dev(ev.rc, np.int32), _dev(ev.depth, np.int16)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, d_depth)
    cat = lambda ch: torch.from_numpy(np.concatenate(ch).astype(np.int32)).cuda()
    keys = mgr(77, chains, cat(join), del_ids=cat(leave), recount=False)
    ids, _ = K.evict_select(keys, ev.k)
    st, state, rc, lat, rkeys, nact = oracle.manager_step(ev.state, ev.rc, ev.lat, ev.depth, 77, chains, join,
                                                          delete=leave, recount=False)
    assert st == oracle.OK
    assert np.array_equal(_u32(d_rc), rc)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
    assert int(mgr.n_active.item()) == nact
    assert np.array_equal(ids.cpu().numpy(), oracle.evict_select(rkeys, ev.k)[1])


def test_manager_invalid_host_chains_change_nothing():
    n = 64
    d_state = torch.zeros(n, dtype=torch.uint8, device="cuda")
    d_lat = torch.zeros(n, dtype=torch.int32, device="cuda")
    d_rc = torch.zeros(n, dtype=torch.int32, device="cuda")
    mgr = K.ManagerStep(d_state, d_rc, d_lat)
    for chains in ([(3, [n])], [(7, [1])], [(3, [-1])]):
        with pytest.raises(K.KvaError) as e:
            mgr(5, chains, None)
        assert e.value.status == K.ERR_INVALID
    torch.cuda.synchronize()
    assert int(d_state.sum()) == 0 and int(d_lat.sum()) == 0


def _thr_workload(types, q_lens, ctx_lens):
    reqs = [W.ReqSpec(t, c, q) for t, q, c in zip(types, q_lens, ctx_lens)]
    return W.make_workload(W.custom_config("thr", 2, 2, 64, 3, reqs, []))


def _append(wl, active, threshold):
    pool = K.Pool(wl.k_pool.cuda(), wl.v_pool.cuda(), K.free_bits_tensor(wl.free_bits, "cuda"))
    pool.set_threshold(threshold)
    pool.set_active_blocks(active)
    batch = K.Batch(wl.batch, "cuda")
    try:
        K.kv_append(pool, batch, wl.k_new.cuda(), wl.v_new.cuda())
        st, deficit = K.OK, 0
    except K.KvaError as e:
        st, deficit = e.status, getattr(e, "deficit", None)
    torch.cuda.synchronize()
    return st, deficit, batch, pool


def test_threshold_parity():
    """S:140-142 / S:171-173 through the library, against the oracle's kv_append_t."""
    wl = _thr_workload([W.ONLINE_DECODE, W.OFFLINE_PREFILL], [1, 64], [33, 64])
    nb = wl.batch["num_blocks"]
    assert nb >= 8
    for active, thr in [(0, nb), (2, 6), (0, 0), (3, 8), (0, -1)]:
        st, deficit, batch, pool = _append(wl, active, thr)
        r = oracle.kv_append(wl.batch, wl.k_pool, wl.v_pool, wl.free_bits, wl.k_new, wl.v_new,
                             active_blocks=active, threshold_blocks=thr)
        assert st == r[0], (active, thr)
        if st == K.NEEDS_EVICTION and deficit is not None:
            assert deficit == r[1]
        assert np.array_equal(batch.table_dev.cpu().numpy(), r[4])
        assert np.array_equal(pool.free_bits.cpu().numpy().view(np.uint32), r[5])
    # online may allocate into the reserve; the same shape offline may not
    for t, expect in [(W.ONLINE_PREFILL, K.OK), (W.OFFLINE_PREFILL, K.NEEDS_EVICTION)]:
        w = _thr_workload([t], [64], [64])
        assert _append(w, 1, 1)[0] == expect


@pytest.mark.parametrize("seed", range(4))
def test_manager_device_resident_chains(seed):
    """kva_manager_update.chains_on_device: the same CSR passed as device arrays gives the
    oracle's state / rc / lat / keys / active count bit-exactly (last chain wins on the device);
    ids outside [0, n) are skipped, i.e. the result equals the oracle on the chains without
    them."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(100, 5000))
    state = rng.integers(0, 6, n).astype(np.uint8)
    lat = rng.integers(0, 100, n).astype(np.uint32)
    depth = rng.integers(0, 8, n).astype(np.uint16)
    rc = np.zeros(n, np.uint32)
    d_state, d_lat, d_rc = _dev(state, np.uint8), _dev(lat, np.int32), _dev(rc, np.int32)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, _dev(depth, np.int16))
    chains = [(int(rng.integers(0, 6)), rng.choice(n, int(rng.integers(1, 40)), replace=False))
              for _ in range(int(rng.integers(1, 12)))]
    bad = [(int(rng.integers(0, 6)), np.concatenate([c[1], [n + 5, -3]])) for c in chains[:1]]
    pool = [rng.choice(n, int(rng.integers(1, 60)), replace=False) for _ in range(int(rng.integers(1, 30)))]
    pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda()
    csr = K.ManagerStep.chains_to_device(K.ManagerStep.chains_csr(bad + chains), "cuda")
    keys = mgr(77, csr, pool_ids)
    torch.cuda.synchronize()
    clean = [(bad[0][0], bad[0][1][:-2])] + chains
    st, state, rc, lat, rkeys, nact = oracle.manager_step(state, rc, lat, depth, 77, clean, pool)
    assert st == oracle.OK
    assert np.array_equal(d_state.cpu().numpy(), state)
    assert np.array_equal(_u32(d_rc), rc) and np.array_equal(_u32(d_lat), lat)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
    assert int(mgr.n_active.item()) == nact


def _fused_select(mgr, now, chains, pool_ids, k, n, **kw):
    ids = torch.full((max(k, 1),), -7, dtype=torch.int32, device="cuda")
    ws = torch.empty(K.evict_select_workspace_size(n, k), dtype=torch.uint8, device="cuda")
    keys = mgr(now, chains, pool_ids, select=(k, ids, ws), **kw)
    torch.cuda.synchronize()
    return keys, ids, int(ws[:8].view(torch.int64).item())


@pytest.mark.parametrize("seed", range(6))
def test_manager_step_select_fused_random(seed):
    """kv_manager_step_select (the manager step and the selection in one kernel) == the oracle's
    manager step then its eviction order, over a sequence of iterations on one workspace (the
    selection's cached layout is exercised across calls); sizes include odd n (scalar slice
    tails) and k above the evictable count."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(50, 40000)) | 1
    state = rng.integers(0, 6, n).astype(np.uint8)
    lat = rng.integers(0, 1 << 20, n).astype(np.uint32)
    depth = rng.integers(0, 64, n).astype(np.uint16)
    rc = np.zeros(n, np.uint32)
    d_state, d_lat, d_rc = _dev(state, np.uint8), _dev(lat, np.int32), _dev(rc, np.int32)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, _dev(depth, np.int16))
    for it in range(3):
        now = (1 << 20) + it
        chains = [(int(rng.integers(0, 6)), rng.choice(n, int(rng.integers(1, 400)), replace=False))
                  for _ in range(int(rng.integers(0, 12)))]
        pool = [rng.choice(n, int(rng.integers(1, 60)), replace=False) for _ in range(int(rng.integers(0, 30)))]
        pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda() if pool else None
        k = int(rng.integers(1, n + 50))
        keys, ids, cnt = _fused_select(mgr, now, chains, pool_ids, k, n)
        st, state, rc, lat, rkeys, nact = oracle.manager_step(state, rc, lat, depth, now, chains, pool)
        assert st == oracle.OK
        assert np.array_equal(d_state.cpu().numpy(), state)
        assert np.array_equal(_u32(d_rc), rc)
        assert np.array_equal(_u32(d_lat), lat)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
        assert int(mgr.n_active.item()) == nact
        _, rids = oracle.evict_select(rkeys, k)
        assert cnt == len(rids)
        assert np.array_equal(ids[:cnt].cpu().numpy(), rids)


@pytest.mark.parametrize("ctas,threads", [(0, 512), (148, 512), (37, 512), (0, 256), (148, 256)])
def test_manager_step_select_fused_full_size(ctas, threads):
    """The `evict` config at full size (2^20 blocks, top-64k), fused, at several grid sizes:
    bit-exact against the oracle."""
    ev = W.make_evict()
    chains, pool = W.make_manager_update(ev, now=1 << 20, seed=1)
    rc0 = np.zeros(len(ev.state), np.uint32)
    d_state, d_lat = _dev(ev.state, np.uint8), _dev(ev.lat, np.int32)
    d_rc, d_depth = _dev(rc0, np.int32), _dev(ev.depth, np.int16)
    mgr = K.ManagerStep(d_state, d_rc, d_lat, d_depth)
    pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda()
    with K.options(evict_ctas=ctas, evict_threads=threads):
        keys, ids, cnt = _fused_select(mgr, 1 << 20, chains, pool_ids, ev.k, len(ev.state))
    st, state, rc, lat, rkeys, nact = oracle.manager_step(ev.state, rc0, ev.lat, ev.depth, 1 << 20, chains, pool)
    assert st == oracle.OK
    assert np.array_equal(_u32(d_rc), rc)
    assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
    assert int(mgr.n_active.item()) == nact
    _, rids = oracle.evict_select(rkeys, ev.k)
    assert cnt == len(rids)
    assert np.array_equal(ids.cpu().numpy(), rids)


def test_manager_step_select_fused_unaligned_metadata():
    """The fused kernel's key pass on metadata views that are not 16-B aligned (every block by
    the scalar path) and an odd block count: bit-exact against the oracle."""
    rng = np.random.default_rng(77)
    n = 20001
    state = rng.integers(0, 6, n + 1).astype(np.uint8)
    lat = rng.integers(0, 1 << 20, n + 1).astype(np.uint32)
    depth = rng.integers(0, 64, n + 1).astype(np.uint16)
    rc = np.zeros(n + 1, np.uint32)
    d_state, d_lat, d_rc = _dev(state, np.uint8)[1:], _dev(lat, np.int32)[1:], _dev(rc, np.int32)[1:]
    d_depth = _dev(depth, np.int16)[1:]
    mgr = K.ManagerStep(d_state, d_rc, d_lat, d_depth)
    st_h, lat_h, dep_h, rc_h = state[1:].copy(), lat[1:].copy(), depth[1:].copy(), rc[1:].copy()
    for it in range(2):
        now = (1 << 20) + it
        chains = [(int(rng.integers(0, 6)), rng.choice(n, int(rng.integers(1, 300)), replace=False)) for _ in range(5)]
        pool = [rng.choice(n, int(rng.integers(1, 60)), replace=False) for _ in range(10)]
        pool_ids = torch.from_numpy(np.concatenate(pool).astype(np.int32)).cuda()
        k = 3000
        keys, ids, cnt = _fused_select(mgr, now, chains, pool_ids, k, n)
        st, st_h, rc_h, lat_h, rkeys, nact = oracle.manager_step(st_h, rc_h, lat_h, dep_h, now, chains, pool)
        assert st == oracle.OK
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), rkeys)
        assert int(mgr.n_active.item()) == nact
        _, rids = oracle.evict_select(rkeys, k)
        assert cnt == len(rids) and np.array_equal(ids[:cnt].cpu().numpy(), rids)
