"""Prefix index + batch grouping, host C++ in libkvattn, against the
brute-force oracle (oracle/prefix.py): SPEC lookup_prefix examples, index
consistency over random operation sequences ("replaying lookup_prefix against a
brute-force longest-common-prefix scan ... gives identical hit_tokens"), grouping of
Table-1-like batches (shared documents, nested system prompt), and an end-to-end check that
the produced groups satisfy the cascade precondition (reading #8) of the oracle's validator."""
import numpy as np
import pytest

import oracle
from oracle.prefix import BruteIndex, group_batch as brute_group, group_batch_nested as oracle_nested
import paper_2504_03651_b200 as K

B = 16


def test_spec_lookup_examples():
    ix = K.PrefixIndex()
    rng = np.random.default_rng(0)
    a = rng.integers(0, 50000, 4 * B)
    ix.insert(a[: 2 * B], [7, 9])
    # S:128 cached chain covers the prompt's first blocks -> exact cover
    assert list(ix.lookup(a)) == [7, 9]
    # S:129 a prompt sharing only 3 tokens with a block -> miss (sub-block prefixes)
    b = a.copy()
    b[3:] = rng.integers(50000, 60000, len(b) - 3)
    assert list(ix.lookup(b)) == []
    # S:130 two groups cached; a prompt from group B returns only group B's chain
    c = rng.integers(60000, 70000, 3 * B)
    ix.insert(c, [11, 12, 13])
    assert list(ix.lookup(np.concatenate([c, a]))) == [11, 12, 13]
    # a different id for a cached block -> INVALID, nothing changed
    with pytest.raises(K.KvaError):
        ix.insert(a[: 2 * B], [7, 99])
    assert ix.size() == 5
    # removing a block drops it and everything below it (no dangling entries)
    ix.remove([12])
    assert list(ix.lookup(c)) == [11] and ix.size() == 3


@pytest.mark.parametrize("seed", range(12))
def test_index_consistency_random_sequences(seed):
    rng = np.random.default_rng(100 + seed)
    ix, ref = K.PrefixIndex(), BruteIndex()
    docs = [rng.integers(0, 1000, int(rng.integers(1, 6)) * B) for _ in range(6)]
    next_id = 0
    resident = []
    for op in range(60):
        r = rng.random()
        if r < 0.45:
            # a prompt = a document prefix (shared) + a private tail
            d = docs[int(rng.integers(0, len(docs)))]
            cut = int(rng.integers(0, len(d) // B + 1)) * B
            tail = rng.integers(1000, 2000, int(rng.integers(0, 4)) * B + int(rng.integers(0, B)))
            toks = np.concatenate([d[:cut], tail]).astype(np.int32)
            hit = list(ix.lookup(toks))
            nb = len(toks) // B
            ids = hit + list(range(next_id, next_id + nb - len(hit)))
            next_id += nb - len(hit)
            ix.insert(toks, ids)
            ref.insert(list(toks), ids)
            resident.extend(ids[len(hit):])
        elif r < 0.6 and resident:
            victims = list(rng.choice(resident, min(len(resident), int(rng.integers(1, 4))), replace=False))
            ix.remove(victims)
            ref.remove(victims)
        q = docs[int(rng.integers(0, len(docs)))]
        q = np.concatenate([q, rng.integers(0, 1000, int(rng.integers(0, 3 * B)))]).astype(np.int32)
        assert list(ix.lookup(q)) == ref.lookup(list(q))
        assert ix.size() == ref.size()


@pytest.mark.parametrize("seed", range(8))
def test_group_batch_random(seed):
    rng = np.random.default_rng(300 + seed)
    ix, ref = K.PrefixIndex(), BruteIndex()
    system = rng.integers(0, 1000, 2 * B)                       # shared by everyone
    docs = [np.concatenate([system, rng.integers(1000, 9000, int(rng.integers(1, 5)) * B)]) for _ in range(4)]
    nid = 0
    for d in docs:                                              # documents resident
        hit = list(ix.lookup(d))
        ids = hit + list(range(nid, nid + len(d) // B - len(hit)))
        nid += len(d) // B - len(hit)
        ix.insert(d, ids)
        ref.insert(list(d), ids)
    reqs = []
    for _ in range(int(rng.integers(2, 20))):
        d = docs[int(rng.integers(0, len(docs)))]
        reqs.append(np.concatenate([d, rng.integers(9000, 9999, int(rng.integers(1, 60)))]).astype(np.int32))
    lim = [int(rng.integers(0, len(r) // B + 1)) for r in reqs]
    for m in (1, 2, 3):
        g1, p1 = ix.group_batch(reqs, lim, min_blocks=m)
        g2, p2 = brute_group(ref, [list(r) for r in reqs], lim, min_blocks=m)
        assert list(g1) == g2 and list(p1) == p2


def test_groups_satisfy_cascade_precondition():
    """Offline tasks sharing a document (LooGLE-like, Table 1): tables built from lookups, groups
    from group_batch -> the oracle's descriptor validation accepts them (reading #8)."""
    rng = np.random.default_rng(7)
    ix = K.PrefixIndex()
    doc_a, doc_b = rng.integers(0, 30000, 8 * B), rng.integers(30000, 60000, 5 * B)
    ix.insert(doc_a, list(range(0, 8)))
    ix.insert(doc_b, list(range(8, 13)))
    nid = 13
    reqs, tables, ctx, ql = [], [], [], []
    for i in range(9):
        d = doc_a if i % 3 else doc_b
        tail = rng.integers(60000, 61000, int(rng.integers(5, 40)))
        t = np.concatenate([d, tail]).astype(np.int32)
        hit = list(ix.lookup(t))
        nb = (len(t) + B - 1) // B
        row = hit + list(range(nid, nid + nb - len(hit)))
        nid += nb - len(hit)
        reqs.append(t)
        tables.append(row)
        ctx.append(len(t))
        ql.append(1)
    lim = [(c - q) // B for c, q in zip(ctx, ql)]
    gof, gpb = ix.group_batch(reqs, lim, min_blocks=1)
    assert len(gpb) == 2 and sorted(set(gof)) == [0, 1]
    mb = max(len(r) for r in tables)
    bt = np.full((len(reqs), mb), -1, np.int32)
    for i, r in enumerate(tables):
        bt[i, : len(r)] = r
    b = dict(num_reqs=len(reqs), num_q_heads=2, num_kv_heads=2, head_dim=64,
             q_indptr=np.concatenate([[0], np.cumsum(ql)]).astype(np.int32),
             ctx_len=np.array(ctx, np.int32), block_table=bt, group_of=gof.astype(np.int32),
             group_prefix_blocks=gpb.astype(np.int32), num_blocks=nid)
    assert oracle.validate(b) == oracle.OK
    assert list(gpb) == [5, 8] or list(gpb) == [8, 5]


@pytest.mark.parametrize("seed", range(6))
def test_group_batch_nested_random(seed):
    """Nested grouping (system prompt -> document -> section) equals the brute-force definition,
    and the output satisfies the descriptor's nesting rules (parents first, longer prefixes)."""
    rng = np.random.default_rng(700 + seed)
    ix, ref = K.PrefixIndex(), BruteIndex()
    system = rng.integers(0, 1000, 2 * B)
    docs = [np.concatenate([system, rng.integers(1000, 9000, int(rng.integers(1, 4)) * B)]) for _ in range(3)]
    secs = [np.concatenate([docs[int(rng.integers(0, 3))], rng.integers(9000, 9500, int(rng.integers(1, 3)) * B)])
            for _ in range(4)]
    nid = 0
    for d in docs + secs:
        hit = list(ix.lookup(d))
        ids = hit + list(range(nid, nid + len(d) // B - len(hit)))
        nid += len(d) // B - len(hit)
        ix.insert(d, ids)
        ref.insert(list(d), ids)
    pool = docs + secs
    reqs = [np.concatenate([pool[int(rng.integers(0, len(pool)))], rng.integers(9900, 9999, int(rng.integers(1, 30)))]).astype(np.int32)
            for _ in range(int(rng.integers(4, 24)))]
    for levels in ([1, 3], [2, 4, 6], [1]):
        g1, p1, a1 = ix.group_batch_nested(reqs, levels)
        g2, p2, a2 = oracle_nested(ref, [list(r) for r in reqs], levels)
        assert list(g1) == g2 and list(p1) == p2 and list(a1) == a2
        for g, (pp, par) in enumerate(zip(p1, a1)):
            assert par < g and (par < 0 or p1[par] < pp)



def test_nested_groups_from_token_ids_match_descriptor():
    """NEXT-3 -> NEXT-4 end to end on the host: token ids of a nested-prefix batch (system prompt
    -> documents) through the prefix index reproduce the descriptor's group_of /
    group_prefix_blocks / group_parent that the GPU multi-level cascade consumes."""
    import workloads as W
    gpb, parent = [6, 14, 10], [-1, 0, 0]
    reqs = []
    for gi in range(3):
        reqs += [W.ReqSpec(W.OFFLINE_DECODE, gpb[gi] * 16 + 5 + j, 1, gi) for j in range(4)]
    wl = W.make_workload(W.custom_config("nest", 4, 2, 64, 5, reqs, gpb, group_parent=parent))
    bt = wl.batch["block_table"]
    tok = lambda blocks: np.repeat(np.asarray(blocks, np.int32) * 7 + 3, B)  # 16 token ids per block
    ix = K.PrefixIndex()
    for gi in range(3):  # the groups' prefix chains are resident (prefix cache)
        first = next(i for i, r in enumerate(reqs) if r.group == gi)
        ix.insert(tok(bt[first, : gpb[gi]]), bt[first, : gpb[gi]])
    toks = [tok(bt[i, : (r.ctx - r.q_len) // B]) for i, r in enumerate(reqs)]
    lim = [(r.ctx - r.q_len) // B for r in reqs]
    gof, p, par = ix.group_batch_nested(toks, [1, 7], lim)
    assert list(gof) == list(wl.batch["group_of"])
    assert list(p) == gpb and list(par) == parent
