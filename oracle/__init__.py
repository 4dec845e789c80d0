"""TEST INFRASTRUCTURE ONLY — the fp64 CPU oracle for the hot path of arxiv 2504.03651.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg
and ``--impl reference``) may import this package.  It shares no code with the CUDA
product in ``paper_2504_03651_b200/``; the only module both sides use is ``workloads``
(seeded input generators, no method arithmetic).

The arithmetic lives in ``oracle.cpp`` (plain C++17, fp64, no -ffast-math); this file
only compiles it with g++ and marshals numpy arrays through ctypes.  Every function
cites the passage it follows (P:n = PAPER.md line n, S:n = SPEC.md line n); readings
of silent passages are listed in DESIGN.md §3.

Parity pins (tests/test_oracle_*.py): dense unpaged numpy attention, torch SDPA fp64,
closed forms (ctx=1, constant V, equal keys), block-permutation / sharing / chunking /
GQA-repeat invariants, brute-force allocation, SPEC eviction examples and a heap free
table with lazy re-insertion.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, INVALID, NEEDS_EVICTION, CAPACITY, EVICTION_SHORT, GROUP = 0, 1, 3, 4, 5, 6

# block states for orc_evict_keys (reading #17)
FREE, RUNNING_ONLINE, PINNED, ACTIVE_OFFLINE, FINISHED_ONLINE, FINISHED_OFFLINE = range(6)


def build(force: bool = False) -> str:
    """Compile oracle.cpp -> liboracle.so with g++ (no CUDA, no fast-math)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                           "-fno-fast-math", "-o", tmp, _SRC])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
            _lib.orc_attention.argtypes = [i32, i32, i32, i32, P, P, P, i32, P, i32, P, i32,
                                           dbl, P, P, P, P, P, ctypes.c_int]
            _lib.orc_attention_rows.argtypes = [i32, i32, i32, i32, P, P, P, i32, P, i32, P, i32,
                                                dbl, P, P, P, P, P, i64, P, P, ctypes.c_int]
            _lib.orc_kv_append.argtypes = [i32, i32, i32, P, P, P, i32, P, i32, P, i32,
                                           P, P, P, P, P, P]
            _lib.orc_kv_append_t.argtypes = [i32, i32, i32, P, P, P, i32, P, i32, P, i32,
                                             P, P, P, P, P, P, P, i64, i64]
            _lib.orc_manager_step.argtypes = [P, P, P, P, i64, ctypes.c_uint32, i32, P, P, P,
                                              i32, P, P, i32, i32, P, P, P, P]
            _lib.orc_evict_keys.argtypes = [P, P, P, P, i64, P]
            _lib.orc_evict_select.argtypes = [P, i64, i64, P, P]
            _lib.orc_evict_select_apply.argtypes = [P, i64, i64, P, P, P]
            _lib.orc_release_blocks.argtypes = [P, i32, P, i64]
            _lib.orc_validate.argtypes = [i32, i32, i32, i32, P, P, P, i32, P, i32, P, i32]
            for f in ("orc_attention", "orc_attention_rows", "orc_kv_append", "orc_kv_append_t",
                      "orc_manager_step", "orc_evict_select_apply", "orc_release_blocks",
                      "orc_evict_keys", "orc_evict_select", "orc_validate"):
                getattr(_lib, f).restype = ctypes.c_int
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def _bits16(t):
    """bf16 tensor/array -> contiguous uint16 numpy array of its bit patterns."""
    try:
        import torch
        if isinstance(t, torch.Tensor):
            t = t.detach().cpu().contiguous()
            if t.dtype == torch.bfloat16:
                t = t.view(torch.int16)
            return t.numpy().view(np.uint16)
    except ImportError:  # pragma: no cover
        pass
    a = np.ascontiguousarray(t)
    return a.view(np.uint16)


def _nthreads(n):
    return int(n) if n else (os.cpu_count() or 1)


def _batch_args(b):
    return (np.int32(b["num_reqs"]), _c(b["q_indptr"], np.int32), _c(b["ctx_len"], np.int32),
            _c(b["block_table"], np.int32), _c(b.get("group_of"), np.int32),
            _c(b.get("group_prefix_blocks"), np.int32))


def attention(b: dict, k_pool, v_pool, q, nthreads: int = 0):
    """Paged causal attention by definition.

    ``b`` keys: num_reqs, num_q_heads, num_kv_heads, head_dim, q_indptr, ctx_len,
    block_table [R][max_blocks], group_of, group_prefix_blocks, num_blocks, sm_scale.
    k_pool/v_pool bf16 [num_blocks][Hkv][16][d]; q bf16 [total_q][Hq][d].
    Returns (status, out fp64 [total_q][Hq][d], lse fp64 [total_q][Hq]).
    """
    lib = _load()
    R, qi, ctx, bt, gof, gpb = _batch_args(b)
    Hq, Hkv, d = b["num_q_heads"], b["num_kv_heads"], b["head_dim"]
    kp, vp, qq = _bits16(k_pool), _bits16(v_pool), _bits16(q)
    total_q = int(qi[-1])
    out = np.zeros((total_q, Hq, d), np.float64)
    lse = np.zeros((total_q, Hq), np.float64)
    st = lib.orc_attention(R, Hq, Hkv, d, _p(qi), _p(ctx), _p(bt), bt.shape[1], _p(gof),
                           len(gpb) if gpb is not None else 0, _p(gpb), b["num_blocks"],
                           float(b.get("sm_scale", 0.0) or 0.0), _p(kp), _p(vp), _p(qq),
                           _p(out), _p(lse), _nthreads(nthreads))
    return st, out, lse


def attention_rows(b: dict, k_pool, v_pool, q, rows, heads, nthreads: int = 0):
    """Sampled (q_row, head) outputs, each exact by definition (rows are independent)."""
    lib = _load()
    R, qi, ctx, bt, gof, gpb = _batch_args(b)
    Hq, Hkv, d = b["num_q_heads"], b["num_kv_heads"], b["head_dim"]
    kp, vp, qq = _bits16(k_pool), _bits16(v_pool), _bits16(q)
    rows = _c(rows, np.int32)
    heads = _c(heads, np.int32)
    n = len(rows)
    out = np.zeros((n, d), np.float64)
    lse = np.zeros((n,), np.float64)
    st = lib.orc_attention_rows(R, Hq, Hkv, d, _p(qi), _p(ctx), _p(bt), bt.shape[1], _p(gof),
                                len(gpb) if gpb is not None else 0, _p(gpb), b["num_blocks"],
                                float(b.get("sm_scale", 0.0) or 0.0), _p(kp), _p(vp), _p(qq),
                                _p(rows), _p(heads), n, _p(out), _p(lse), _nthreads(nthreads))
    return st, out, lse


def kv_append(b: dict, k_pool, v_pool, free_bits, k_new, v_new, active_blocks=0, threshold_blocks=-1):
    """KV append + smallest-free-id allocation (Eq.(5)), with the
    optional burst-reserve threshold (offline allocations may not push
    the active classes over threshold_blocks, online ones may use the reserve).

    Works on copies; returns (status, deficit, k_pool', v_pool', block_table', free_bits')
    with the pools as uint16 bit arrays.
    """
    lib = _load()
    if threshold_blocks >= 0:
        R, qi, ctx, bt, gof, gpb = _batch_args(b)
        bt = bt.copy()
        Hkv, d = b["num_kv_heads"], b["head_dim"]
        kp, vp = _bits16(k_pool).copy(), _bits16(v_pool).copy()
        fb = _c(free_bits, np.uint32).copy()
        kn, vn = _bits16(k_new), _bits16(v_new)
        rt = _c(b["req_type"], np.int32)
        deficit = np.zeros(1, np.int32)
        st = lib.orc_kv_append_t(R, Hkv, d, _p(qi), _p(ctx), _p(bt), bt.shape[1], _p(gof),
                                 len(gpb) if gpb is not None else 0, _p(gpb), b["num_blocks"],
                                 _p(kp), _p(vp), _p(fb), _p(kn), _p(vn), _p(deficit), _p(rt),
                                 int(active_blocks), int(threshold_blocks))
        return st, int(deficit[0]), kp, vp, bt, fb
    R, qi, ctx, bt, gof, gpb = _batch_args(b)
    bt = bt.copy()
    Hkv, d = b["num_kv_heads"], b["head_dim"]
    kp, vp = _bits16(k_pool).copy(), _bits16(v_pool).copy()
    fb = _c(free_bits, np.uint32).copy()
    kn, vn = _bits16(k_new), _bits16(v_new)
    deficit = np.zeros(1, np.int32)
    st = lib.orc_kv_append(R, Hkv, d, _p(qi), _p(ctx), _p(bt), bt.shape[1], _p(gof),
                           len(gpb) if gpb is not None else 0, _p(gpb), b["num_blocks"],
                           _p(kp), _p(vp), _p(fb), _p(kn), _p(vn), _p(deficit))
    return st, int(deficit[0]), kp, vp, bt, fb


def evict_keys(state, rc, lat, depth=None):
    """priority_of as order-preserving u64 keys (readings #15-#20)."""
    lib = _load()
    st_ = _c(state, np.uint8)
    rc_ = _c(rc, np.uint32)
    lat_ = _c(lat, np.uint32)
    dep = _c(depth, np.uint16)
    n = len(st_)
    keys = np.zeros(n, np.uint64)
    s = lib.orc_evict_keys(_p(st_), _p(rc_), _p(lat_), _p(dep), n, _p(keys))
    return s, keys


def _csr(chains):
    ip = np.zeros(len(chains) + 1, np.int32)
    for j, ids in enumerate(chains):
        ip[j + 1] = ip[j] + len(ids)
    flat = np.concatenate([np.asarray(ids, np.int32) for ids in chains]) if chains else np.zeros(0, np.int32)
    return ip, flat


def manager_step(state, rc, lat, depth, now, chains, pool, delete=None, recount=True):
    """The KV manager's per-iteration metadata pass:
    class transitions (chains = [(state, ids), ...], in order, lat = now), reference counts
    (recount=True: rc = #pool chains listing the block; recount=False: rc += #chains of `pool`
    (joined) - #chains of `delete` (left)), active-class count, eviction keys.
    Works on copies; returns (status, state', rc', lat', keys, n_active)."""
    lib = _load()
    st_ = _c(state, np.uint8).copy()
    rc_ = np.zeros(len(st_), np.uint32) if rc is None else _c(rc, np.uint32).copy()
    lat_ = _c(lat, np.uint32).copy()
    dep = _c(depth, np.uint16)
    ci = np.zeros(len(chains) + 1, np.int32)
    for j, (_, ids) in enumerate(chains):
        ci[j + 1] = ci[j] + len(ids)
    cids = np.concatenate([np.asarray(ids, np.int32) for _, ids in chains]) if chains else np.zeros(0, np.int32)
    cst = np.array([s_ for s_, _ in chains], np.uint8)
    pi, pids = _csr(pool)
    delete = delete or []
    di, dids = _csr(delete)
    n = len(st_)
    keys = np.zeros(n, np.uint64)
    nact = np.zeros(1, np.int64)
    s = lib.orc_manager_step(_p(st_), _p(rc_), _p(lat_), _p(dep), n, int(now) & 0xFFFFFFFF,
                             len(chains), _p(ci), _p(cids), _p(cst), len(pool), _p(pi), _p(pids),
                             1 if recount else 0, len(delete), _p(di), _p(dids), _p(keys), _p(nact))
    return s, st_, rc_, lat_, keys, int(nact[0])


def evict_select(keys, k: int):
    """Eviction order: (key, id) ascending, first k."""
    lib = _load()
    kk = _c(keys, np.uint64)
    out = np.full(max(int(k), 0), -1, np.int32)
    nsel = np.zeros(1, np.int64)
    s = lib.orc_evict_select(_p(kk), len(kk), int(k), _p(out), _p(nsel))
    return s, out[: int(nsel[0])]


def evict_select_apply(keys, k: int, free_bits):
    """evict_select with apply: the same order, then the selected
    blocks' free bits are set.  Works on a copy; returns (status, ids, free_bits')."""
    lib = _load()
    kk = _c(keys, np.uint64)
    out = np.full(max(int(k), 0), -1, np.int32)
    nsel = np.zeros(1, np.int64)
    fb = _c(free_bits, np.uint32).copy()
    assert len(fb) >= (len(kk) + 31) // 32
    s = lib.orc_evict_select_apply(_p(kk), len(kk), int(k), _p(out), _p(nsel), _p(fb))
    return s, out[: int(nsel[0])], fb


def release_blocks(free_bits, num_blocks: int, ids):
    """Return blocks to the free pool: each id allocated and listed once,
    else INVALID with nothing changed.  Works on a copy; returns (status, free_bits')."""
    lib = _load()
    fb = _c(free_bits, np.uint32).copy()
    ii = _c(ids, np.int32)
    s = lib.orc_release_blocks(_p(fb), int(num_blocks), _p(ii), len(ii))
    return s, fb


def truncate(b: dict, free_bits, keep_len):
    """Shorten request i to its first keep_len[i] tokens ("preempts and release the KV
    cache of the victim request"; -1 = untouched): the non-(-1) table entries of row i at block
    indices [ceil(keep/16), ceil(ctx/16)) are released (release_blocks: allocated, each once)
    and set to -1.  A cut inside the request's group prefix is GROUP; a keep_len outside
    [0, ctx] is INVALID.  Works on copies; returns (status, free_bits', block_table')."""
    bt = np.array(b["block_table"], np.int32, copy=True)
    fb = _c(free_bits, np.uint32).copy()
    gof, gpb = b.get("group_of"), b.get("group_prefix_blocks")
    ids, ent = [], []
    for i, keep in enumerate(np.asarray(keep_len, np.int64)):
        if keep == -1:
            continue
        ctx = int(b["ctx_len"][i])
        if keep < 0 or keep > ctx:
            return INVALID, fb, bt
        k0 = -(-int(keep) // 16)
        if gof is not None and gof[i] >= 0 and k0 < int(gpb[gof[i]]):
            return GROUP, fb, bt
        for k in range(k0, -(-ctx // 16)):
            if bt[i, k] != -1:
                ids.append(int(bt[i, k]))
                ent.append((i, k))
    s, fb2 = release_blocks(fb, b["num_blocks"], np.array(ids, np.int32))
    if s != OK:
        return s, fb, bt
    for i, k in ent:
        bt[i, k] = -1
    return OK, fb2, bt


def validate(b: dict):
    lib = _load()
    R, qi, ctx, bt, gof, gpb = _batch_args(b)
    return lib.orc_validate(R, b["num_q_heads"], b["num_kv_heads"], b["head_dim"], _p(qi),
                            _p(ctx), _p(bt), bt.shape[1], _p(gof),
                            len(gpb) if gpb is not None else 0, _p(gpb), b["num_blocks"])
