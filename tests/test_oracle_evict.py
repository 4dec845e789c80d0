"""Pins for the eviction oracle (priority_of + order), SURVEY §8(c) c3.

* SPEC/paper examples (tests/golden/spec_evict_examples.json, each cited).
* A heap free table with lazy re-insertion keyed by Python tuples
  (priority as a real number with inf, lat, -depth, id) — an encoding independent of the
  oracle's u64 keys — over 1,000 random operation sequences: every eviction must
  pick the same blocks in the same order.
* Invariants: victim optimality, no inf block ever selected, SHORT when
  fewer than k are evictable, depth=None reduces to (priority, lat, id).
"""
import heapq
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_evict_examples.json")
INF = UINT64_MAX = np.uint64(0xFFFFFFFFFFFFFFFF)


def _priority(state, rc):
    """P:331-334 restated with real numbers (readings #15-#17)."""
    if state in (0, 1, 2):
        return math.inf
    if rc > 0:
        return float(rc)
    return 0.5 if state == 4 else 0.0


def test_golden_priority_examples():
    gold = json.load(open(GOLD))
    for ex in gold["priority_of"]:
        st, keys = oracle.evict_keys([ex["state"]], [ex["rc"]], [0], None)
        assert st == oracle.OK
        if ex.get("key_is_inf"):
            assert keys[0] == UINT64_MAX, ex["cite"]
        else:
            assert int(keys[0]) >> 48 == ex["code"], ex["cite"]


def test_golden_evict_examples():
    gold = json.load(open(GOLD))
    for ex in gold["evict"]:
        bl = ex["blocks"]
        st, keys = oracle.evict_keys([b["state"] for b in bl], [b["rc"] for b in bl],
                                     [b["lat"] for b in bl], None)
        s, ids = oracle.evict_select(keys, ex["k"])
        assert list(ids) == ex["expect"], ex["cite"]
        assert s == (oracle.EVICTION_SHORT if ex.get("short") else oracle.OK), ex["cite"]


def test_depth_tiebreak_and_null_depth():
    # equal (priority, lat): deepest block of a chain first (reading #19), then id
    st, keys = oracle.evict_keys([5, 5, 5], [0, 0, 0], [7, 7, 7], [0, 3, 3])
    assert list(oracle.evict_select(keys, 3)[1]) == [1, 2, 0]
    st, keys = oracle.evict_keys([5, 5, 5], [0, 0, 0], [7, 7, 7], None)
    assert list(oracle.evict_select(keys, 3)[1]) == [0, 1, 2]


def test_rc_saturation_and_invalid_state():
    st, keys = oracle.evict_keys([3, 3], [40000, 32767], [0, 0], None)
    assert int(keys[0]) >> 48 == 0xFFFE and int(keys[1]) >> 48 == 0xFFFE
    assert keys[0] != UINT64_MAX
    st, _ = oracle.evict_keys([9], [0], [0], None)
    assert st == oracle.INVALID


class HeapFreeTable:
    """priority queue keyed by (priority, lat, -depth, id); lazy re-insertion."""

    def __init__(self, state, rc, lat, depth):
        self.state, self.rc, self.lat, self.depth = state, rc, lat, depth
        self.h = []
        for b in range(len(state)):
            self.push(b)

    def cur(self, b):
        return (_priority(self.state[b], self.rc[b]), int(self.lat[b]), -int(self.depth[b]), b)

    def push(self, b):
        e = self.cur(b)
        if e[0] != math.inf:
            heapq.heappush(self.h, e)

    def evict(self, k):
        out = []
        while self.h and len(out) < k:
            e = heapq.heappop(self.h)
            if e != self.cur(e[3]) or e[3] in out:
                continue  # stale entry
            out.append(e[3])
        return out


def test_heap_free_table_random_sequences():
    rng = np.random.default_rng(590)
    for seq in range(1000):
        n = int(rng.integers(1, 48))
        state = rng.integers(0, 6, n).astype(np.uint8)
        rc = np.where(rng.random(n) < 0.5, rng.integers(0, 5, n), 0).astype(np.uint32)
        lat = rng.integers(0, 8, n).astype(np.uint32)
        depth = rng.integers(0, 4, n).astype(np.uint16)
        heap = HeapFreeTable(state, rc, lat, depth)
        now = 8
        for op in range(int(rng.integers(1, 8))):
            kind = rng.integers(0, 3)
            if kind == 0:   # touch a few blocks (LAT refresh) or reclass them
                for b in rng.integers(0, n, int(rng.integers(1, 4))):
                    lat[b] = now
                    if rng.random() < 0.3:
                        state[b] = rng.integers(1, 6)
                        rc[b] = rng.integers(0, 4) if rng.random() < 0.5 else 0
                    heap.push(int(b))
                now += 1
            else:           # evict k blocks
                k = int(rng.integers(0, n + 2))
                expect = heap.evict(k)
                st, keys = oracle.evict_keys(state, rc, lat, depth)
                assert st == oracle.OK
                s, got = oracle.evict_select(keys, k)
                assert list(got) == expect, (seq, op)
                assert s == (oracle.OK if len(expect) == k else oracle.EVICTION_SHORT)
                # victim optimality + no inf
                sel = set(got.tolist())
                ev = [b for b in range(n) if keys[b] != UINT64_MAX]
                if got.size:
                    worst = max((keys[b], b) for b in got)
                    for b in ev:
                        if b not in sel:
                            assert (keys[b], b) > worst
                assert all(keys[b] != UINT64_MAX for b in got)
                for b in got:   # apply: evicted blocks become free
                    state[b] = 0
                    rc[b] = 0


def test_large_select_matches_heap():
    import workloads as W
    ev = W.make_evict(n=1 << 14, k=1 << 10, seed=5)
    st, keys = oracle.evict_keys(ev.state, ev.rc, ev.lat, ev.depth)
    assert st == oracle.OK
    s, got = oracle.evict_select(keys, ev.k)
    heap = HeapFreeTable(ev.state, ev.rc, ev.lat, ev.depth)
    assert list(got) == heap.evict(ev.k)


def _bits_of(fb, n):
    return {b for b in range(n) if (int(fb[b // 32]) >> (b % 32)) & 1}


@pytest.mark.parametrize("seed", range(5))
def test_evict_apply_sets_exactly_the_victims_free(seed):
    """SURVEY c1.4 apply (P:440 the victims return to the free table; S:146 removed): the free
    set afterwards is the free set before plus exactly the selected ids — set arithmetic on
    Python sets, with the selection itself pinned by the heap free table above."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 3000))
    state = rng.integers(0, 6, n).astype(np.uint8)
    rc = np.where(rng.random(n) < 0.3, rng.integers(1, 5, n), 0).astype(np.uint32)
    lat = rng.integers(0, 20, n).astype(np.uint32)
    fb = np.zeros((n + 31) // 32, np.uint32)
    for b in range(n):
        if state[b] == 0:
            fb[b // 32] |= np.uint32(1 << (b % 32))
    _, keys = oracle.evict_keys(state, rc, lat, None)
    k = int(rng.integers(0, n + 5))
    s, ids = oracle.evict_select(keys, k)
    s2, ids2, fb2 = oracle.evict_select_apply(keys, k, fb)
    assert s2 == s and list(ids2) == list(ids)
    before = {b for b in range(n) if state[b] == 0}
    assert _bits_of(fb2, n) == before | set(ids.tolist())
    assert not (before & set(ids.tolist()))   # a free block is never a victim (key inf)
    assert len(_bits_of(fb2, n)) == len(before) + len(ids)


def test_release_blocks_oracle():
    """P:448 release / S:143-146: allocated ids become free; a free, duplicated or
    out-of-range id is INVALID and changes nothing."""
    n = 70
    fb = np.zeros(3, np.uint32)
    fb[0] = 0x0000FFFF            # blocks 0..15 free
    s, fb2 = oracle.release_blocks(fb, n, [20, 69, 16])
    assert s == oracle.OK and _bits_of(fb2, n) == set(range(16)) | {16, 20, 69}
    for bad in ([3], [20, 20], [70], [-1], [21, 5]):
        s, fb3 = oracle.release_blocks(fb, n, bad)
        assert s == oracle.INVALID and np.array_equal(fb3, fb), bad
    s, fb4 = oracle.release_blocks(fb, n, [])
    assert s == oracle.OK and np.array_equal(fb4, fb)


def test_truncate_oracle_roundtrip_and_errors():
    """kv_truncate's oracle (P:448 release of a victim's KV): after kv_append, truncating every
    request to its pre-append length restores the pristine table and free bitmap exactly (the
    inverse of the append's allocation); keep = ctx is a no-op; keep = 0 on an ungrouped
    request frees its whole row; a cut inside a group prefix is GROUP, keep > ctx INVALID,
    and neither changes anything."""
    import workloads as W
    wl = W.make_workload("tiny")
    b = wl.batch
    s, _, _, _, bt, fb = oracle.kv_append(b, wl.k_pool, wl.v_pool, wl.free_bits, wl.k_new, wl.v_new)
    assert s == oracle.OK
    b2 = dict(b, block_table=bt)
    ql = np.diff(b["q_indptr"])
    keep = (b["ctx_len"] - ql).astype(np.int32)
    s, fb_t, bt_t = oracle.truncate(b2, fb, keep)
    assert s == oracle.OK
    assert np.array_equal(bt_t, b["block_table"]) and np.array_equal(fb_t, wl.free_bits)
    s, fb_n, bt_n = oracle.truncate(b2, fb, b["ctx_len"])
    assert s == oracle.OK and np.array_equal(bt_n, bt) and np.array_equal(fb_n, fb)
    n = b["num_blocks"]
    gof = b["group_of"]
    i = int(np.nonzero(gof < 0)[0][0])
    keep0 = np.full(len(keep), -1, np.int32)
    keep0[i] = 0
    s, fb0, bt0 = oracle.truncate(b2, fb, keep0)
    row = {int(x) for x in bt[i] if x >= 0}
    assert s == oracle.OK and _bits_of(fb0, n) == _bits_of(fb, n) | row and (bt0[i] == -1).all()
    assert np.array_equal(np.delete(bt0, i, 0), np.delete(bt, i, 0))
    j = int(np.nonzero(gof >= 0)[0][0])
    bad = np.full(len(keep), -1, np.int32)
    bad[j] = 16 * (int(b["group_prefix_blocks"][gof[j]]) - 1)  # releases the last prefix block
    s, fbx, btx = oracle.truncate(b2, fb, bad)
    assert s == oracle.GROUP and np.array_equal(fbx, fb) and np.array_equal(btx, bt)
    bad[j] = int(b["ctx_len"][j]) + 1
    s, fbx, btx = oracle.truncate(b2, fb, bad)
    assert s == oracle.INVALID and np.array_equal(fbx, fb) and np.array_equal(btx, bt)
