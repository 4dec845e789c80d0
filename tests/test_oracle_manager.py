"""Pins for the KV-manager step oracle (§4.2) and
the burst-reserve threshold of kv_append.

* SPEC examples, each cited: update_references, release_request,
  allocate with the threshold, set_threshold boundaries.
* Brute force: an independent pure-Python manager (dicts and sets, priorities as real
  numbers with inf, order by Python tuples) replayed over random operation sequences; the
  oracle's state, rc, lat, active count and eviction order must match it exactly.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as W

FREE, RUN_ON, PINNED, ACT_OFF, FIN_ON, FIN_OFF = range(6)


def _code(keys, b):
    return int(keys[b]) >> 48


def test_update_references_examples():
    n = 400
    state = np.full(n, FIN_OFF, np.uint8)
    lat = np.zeros(n, np.uint32)
    prefix = list(range(10, 10 + 128))  # one 2048-token prefix = 128 blocks of 16
    # S:158 "3 pool requests share one 2048-token prefix -> each covering block has rc=3"
    st, s2, rc, l2, keys, nact = oracle.manager_step(state, None, lat, None, 1, [], [prefix] * 3)
    assert st == oracle.OK
    assert all(rc[b] == 3 for b in prefix) and rc.sum() == 3 * 128
    assert all(_code(keys, b) == 6 for b in prefix)          # priority rc = 3 -> code 6
    assert nact == 128                                        # ActiveOffline
    # S:159 "request finishes and leaves pool -> rc decremented on its chain"
    st, _, rc, _, keys, _ = oracle.manager_step(state, None, lat, None, 2, [], [prefix] * 2)
    assert all(rc[b] == 2 for b in prefix)
    # S:160 "disjoint prompts -> all rc <= 1"
    pool = [list(range(i * 20, i * 20 + 20)) for i in range(5)]
    st, _, rc, _, _, nact = oracle.manager_step(state, None, lat, None, 3, [], pool)
    assert rc.max() == 1 and rc.sum() == 100 and nact == 100


def test_release_request_examples():
    n = 64
    state = np.full(n, FREE, np.uint8)
    lat = np.zeros(n, np.uint32)
    a, b, c = list(range(0, 8)), list(range(8, 16)), list(range(16, 24))
    # the three requests run: online a (running online), offline b and c (pinned while in batch)
    st, state, rc, lat, keys, nact = oracle.manager_step(
        state, None, lat, None, 5, [(RUN_ON, a), (PINNED, b), (PINNED, c)], [b, c])
    assert st == oracle.OK and nact == 24
    assert all(keys[i] == np.uint64(0xFFFFFFFFFFFFFFFF) for i in a + b + c)   # P:331 "priority=inf"
    # S:166 finished online -> FinishedOnline, priority 0.5
    # S:167 preempted offline, no other sharers -> ActiveOffline rc=1 (its own pool entry)
    # S:168 finished offline, rc becomes 0 -> priority 0
    st, state, rc, lat, keys, nact = oracle.manager_step(
        state, rc, lat, None, 9, [(FIN_ON, a), (ACT_OFF, b), (FIN_OFF, c)], [b])
    assert st == oracle.OK
    assert all(_code(keys, i) == 1 for i in a)
    assert all(rc[i] == 1 and _code(keys, i) == 2 for i in b)
    assert all(rc[i] == 0 and _code(keys, i) == 0 for i in c)
    assert all(lat[i] == 9 for i in a + b + c)
    assert nact == 8                                           # only b stays active
    # eviction order: priority dominates recency: c (0) before a (0.5) before b (1)
    s, ids = oracle.evict_select(keys, 24)
    assert list(ids[:8]) == c and list(ids[8:16]) == a and list(ids[16:]) == b


def test_transition_order_and_validation():
    n = 16
    state = np.full(n, FIN_OFF, np.uint8)
    lat = np.zeros(n, np.uint32)
    # a later chain overrides an earlier one (the caller lists this iteration's pins last)
    st, s2, _, _, keys, _ = oracle.manager_step(state, None, lat, None, 4, [(FIN_ON, [1, 2]), (PINNED, [2])], [])
    assert st == oracle.OK and s2[1] == FIN_ON and s2[2] == PINNED
    # invalid id / state / indptr -> INVALID, inputs untouched (the wrapper works on copies;
    # the C function validates before writing)
    for chains, pool in [([(FIN_ON, [16])], []), ([(9, [1])], []), ([], [[-1]])]:
        st, s3, _, l3, _, _ = oracle.manager_step(state, None, lat, None, 4, chains, pool)
        assert st == oracle.INVALID
        assert np.array_equal(s3, state) and np.array_equal(l3, lat)


# ------------------------------------------------------------------------------------------
# independent brute-force manager (sets, real priorities, Python tuples)
class RefManager:
    def __init__(self, n, rng):
        self.cls = {b: int(rng.choice([FREE, FIN_ON, FIN_OFF, ACT_OFF])) for b in range(n)}
        self.lat = {b: int(rng.integers(0, 50)) for b in range(n)}
        self.depth = {b: int(rng.integers(0, 5)) for b in range(n)}

    def step(self, now, chains, pool):
        for st, ids in chains:
            for b in ids:
                self.cls[b] = st
                self.lat[b] = now
        self.rc = {b: sum(1 for p in pool for x in p if x == b) for b in self.cls}
        act = sum(1 for b, c in self.cls.items()
                  if c != FREE and (c in (RUN_ON, PINNED) or self.rc[b] > 0))
        return act

    def priority(self, b):
        c = self.cls[b]
        if c in (FREE, RUN_ON, PINNED):
            return math.inf
        if self.rc[b] > 0:
            return float(self.rc[b])
        return 0.5 if c == FIN_ON else 0.0

    def order(self):
        ev = [b for b in self.cls if self.priority(b) != math.inf]
        return sorted(ev, key=lambda b: (self.priority(b), self.lat[b], -self.depth[b], b))


@pytest.mark.parametrize("seed", range(40))
def test_manager_bruteforce_sequences(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(20, 120))
    ref = RefManager(n, rng)
    state = np.array([ref.cls[b] for b in range(n)], np.uint8)
    lat = np.array([ref.lat[b] for b in range(n)], np.uint32)
    depth = np.array([ref.depth[b] for b in range(n)], np.uint16)
    rc = np.zeros(n, np.uint32)
    for it in range(6):
        now = 100 + it
        chains = [(int(rng.integers(0, 6)), list(rng.choice(n, int(rng.integers(1, 10)), replace=False)))
                  for _ in range(int(rng.integers(0, 6)))]
        pool = [list(rng.choice(n, int(rng.integers(1, 15)), replace=False))
                for _ in range(int(rng.integers(0, 8)))]
        act = ref.step(now, chains, pool)
        st, state, rc, lat, keys, nact = oracle.manager_step(state, rc, lat, depth, now, chains, pool)
        assert st == oracle.OK
        assert [int(x) for x in state] == [ref.cls[b] for b in range(n)]
        assert [int(x) for x in rc] == [ref.rc[b] for b in range(n)]
        assert [int(x) for x in lat] == [ref.lat[b] for b in range(n)]
        assert nact == act
        k = int(rng.integers(1, n + 1))
        s, ids = oracle.evict_select(keys, k)
        exp = ref.order()
        assert list(ids) == exp[:k]
        assert s == (oracle.EVICTION_SHORT if len(exp) < k else oracle.OK)


# ------------------------------------------------------------------------------------------
# burst-reserve threshold in kv_append
def _small_batch(types, q_lens, ctx_lens, seed=3):
    reqs = [W.ReqSpec(t, c, q) for t, q, c in zip(types, q_lens, ctx_lens)]
    return W.make_workload(W.custom_config("thr", 2, 2, 64, seed, reqs, []))


def test_threshold_examples():
    # one online decode needing a new block + one offline prefill needing 4 new blocks
    wl = _small_batch([W.ONLINE_DECODE, W.OFFLINE_PREFILL], [1, 64], [33, 64])
    b = wl.batch
    args = (wl.k_pool, wl.v_pool, wl.free_bits, wl.k_new, wl.v_new)
    st0, _, kp0, vp0, bt0, fb0 = oracle.kv_append(b, *args)
    assert st0 == oracle.OK
    need = int(((bt0 >= 0) & (b["block_table"] == -1)).sum())
    assert need == 5
    nb = b["num_blocks"]
    # S:140 ample space, no threshold -> granted; threshold = capacity disables the reserve
    # ("tokens = capacity -> reserve disabled (Fig. 5(a))"): identical result
    st, _, kp, vp, bt, fb = oracle.kv_append(b, *args, active_blocks=0, threshold_blocks=nb)
    assert st == oracle.OK and np.array_equal(bt, bt0) and np.array_equal(fb, fb0)
    # S:141 offline allocation exceeding the threshold but not capacity -> NeedsEviction,
    # state unchanged
    st, deficit, kp, vp, bt, fb = oracle.kv_append(b, *args, active_blocks=10, threshold_blocks=12)
    assert st == oracle.NEEDS_EVICTION and deficit == 10 + 5 - 12
    assert np.array_equal(bt, b["block_table"]) and np.array_equal(fb, wl.free_bits)
    # S:142 online allocation into the reserve above the threshold -> granted; offline with
    # the identical shape -> rejected
    won = _small_batch([W.ONLINE_PREFILL], [64], [64])
    woff = _small_batch([W.OFFLINE_PREFILL], [64], [64])
    st_on = oracle.kv_append(won.batch, won.k_pool, won.v_pool, won.free_bits, won.k_new, won.v_new,
                             active_blocks=12, threshold_blocks=12)[0]
    st_off = oracle.kv_append(woff.batch, woff.k_pool, woff.v_pool, woff.free_bits, woff.k_new, woff.v_new,
                              active_blocks=12, threshold_blocks=12)[0]
    assert st_on == oracle.OK and st_off == oracle.NEEDS_EVICTION
    # S:173 "tokens = 0 -> all offline allocations rejected"
    assert oracle.kv_append(woff.batch, woff.k_pool, woff.v_pool, woff.free_bits, woff.k_new, woff.v_new,
                            active_blocks=0, threshold_blocks=0)[0] == oracle.NEEDS_EVICTION
    # capacity is checked first: more than the free blocks -> deficit vs free blocks
    fb_small = wl.free_bits.copy()
    free = [i for i in range(nb) if (int(fb_small[i // 32]) >> (i % 32)) & 1]
    for i in free[2:]:
        fb_small[i // 32] &= ~np.uint32(1 << (i % 32))
    st, deficit = oracle.kv_append(b, wl.k_pool, wl.v_pool, fb_small, wl.k_new, wl.v_new,
                                   active_blocks=0, threshold_blocks=nb)[:2]
    assert st == oracle.NEEDS_EVICTION and deficit == 3


@pytest.mark.parametrize("seed", range(10))
def test_incremental_counts_equal_recount(seed):
    """Incremental mode (requests joining / leaving the offline pool) must equal a full recount
    of the new pool ("request finishes and leaves pool -> rc decremented")."""
    rng = np.random.default_rng(77 + seed)
    n = int(rng.integers(30, 300))
    state = rng.integers(0, 6, n).astype(np.uint8)
    lat = rng.integers(0, 9, n).astype(np.uint32)
    pool = [list(rng.choice(n, int(rng.integers(1, 20)), replace=False)) for _ in range(int(rng.integers(1, 25)))]
    st, s1, rc1, l1, _, _ = oracle.manager_step(state, None, lat, None, 3, [], pool)
    leave = sorted(set(rng.choice(len(pool), int(rng.integers(0, len(pool) + 1)), replace=False).tolist()))
    join = [list(rng.choice(n, int(rng.integers(1, 20)), replace=False)) for _ in range(int(rng.integers(0, 10)))]
    new_pool = [p for i, p in enumerate(pool) if i not in leave] + join
    st_a, sa, rca, la, ka, na = oracle.manager_step(s1, rc1, l1, None, 4, [], join,
                                                    delete=[pool[i] for i in leave], recount=False)
    st_b, sb, rcb, lb, kb, nb = oracle.manager_step(s1, rc1, l1, None, 4, [], new_pool)
    assert st_a == st_b == oracle.OK
    assert np.array_equal(rca, rcb) and np.array_equal(ka, kb) and na == nb
    # a count would go negative -> INVALID, nothing changed
    st_c, sc, rcc, _, _, _ = oracle.manager_step(s1, np.zeros(n, np.uint32), l1, None, 4, [], [],
                                                 delete=[pool[0]], recount=False)
    assert st_c == oracle.INVALID and not rcc.any()
