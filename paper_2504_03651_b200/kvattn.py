"""Thin ctypes binding of libkvattn.so (include/kvattn.h) — argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; PyTorch only supplies
device memory, streams and (in bench.py) process groups.  There is no CPU fallback: if the
library is missing or CUDA is unavailable, these functions raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _build

OK, ERR_INVALID, ERR_UNSUPPORTED, NEEDS_EVICTION, ERR_CAPACITY, EVICTION_SHORT, ERR_GROUP, ERR_CUDA = range(8)
OUT_BF16, OUT_F32 = 0, 1
STATUS_NAMES = {0: "OK", 1: "ERR_INVALID", 2: "ERR_UNSUPPORTED", 3: "NEEDS_EVICTION",
                4: "ERR_CAPACITY", 5: "EVICTION_SHORT", 6: "ERR_GROUP", 7: "ERR_CUDA"}


class KvaError(RuntimeError):
    def __init__(self, status, msg, **extra):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.__dict__.update(extra)


class PoolDesc(ctypes.Structure):
    _fields_ = [("num_blocks", ctypes.c_int32), ("block_size", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("k_pool", ctypes.c_void_p), ("v_pool", ctypes.c_void_p),
                ("free_bits", ctypes.c_void_p), ("device", ctypes.c_int32)]


class BatchDesc(ctypes.Structure):
    _fields_ = [("num_reqs", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("req_type", ctypes.c_void_p), ("q_indptr", ctypes.c_void_p),
                ("ctx_len", ctypes.c_void_p), ("block_table", ctypes.c_void_p),
                ("block_table_host", ctypes.c_void_p), ("max_blocks", ctypes.c_int32),
                ("group_of", ctypes.c_void_p), ("num_groups", ctypes.c_int32),
                ("group_prefix_blocks", ctypes.c_void_p), ("sm_scale", ctypes.c_float),
                ("group_parent", ctypes.c_void_p)]


class BlockMeta(ctypes.Structure):
    _fields_ = [("num_blocks", ctypes.c_int64), ("state", ctypes.c_void_p), ("rc", ctypes.c_void_p),
                ("lat", ctypes.c_void_p), ("depth", ctypes.c_void_p)]


class ManagerUpdate(ctypes.Structure):
    _fields_ = [("now", ctypes.c_uint32), ("n_chains", ctypes.c_int32), ("chain_indptr", ctypes.c_void_p),
                ("chain_ids", ctypes.c_void_p), ("chain_state", ctypes.c_void_p), ("recount", ctypes.c_int32),
                ("pool_ids", ctypes.c_void_p), ("pool_len", ctypes.c_int64), ("del_ids", ctypes.c_void_p),
                ("del_len", ctypes.c_int64), ("chains_on_device", ctypes.c_int32), ("n_chain_ids", ctypes.c_int64)]


class PlanStats(ctypes.Structure):
    _fields_ = [("n_decode_items", ctypes.c_int64), ("n_tile_items", ctypes.c_int64),
                ("n_cascade_items", ctypes.c_int64), ("n_merge_rows", ctypes.c_int64),
                ("kv_bytes_algorithmic", ctypes.c_int64), ("q_bytes", ctypes.c_int64),
                ("o_bytes", ctypes.c_int64), ("decode_kv_bytes", ctypes.c_int64),
                ("flops", ctypes.c_int64), ("tile_flops", ctypes.c_int64),
                ("host_validate_ns", ctypes.c_int64), ("host_build_ns", ctypes.c_int64),
                ("host_total_ns", ctypes.c_int64)]


EXPORTS = ["kva_last_error", "kva_version", "kva_validate_batch", "kv_pool_create", "kv_pool_destroy",
           "kv_pool_free_count", "kv_pool_resync", "kv_pool_sync", "kv_append_workspace_size", "kv_append",
           "hybrid_attention_workspace_size", "hybrid_attention_plan", "kv_append_plan", "hybrid_attention_run",
           "hybrid_attention_run_phases", "kva_plan_launch_count", "kva_plan_set_timing_events",
           "kva_plan_set_span_buffer", "kva_plan_set_outputs",
           "kva_plan_destroy",
           "kva_plan_get_stats", "hybrid_attention", "kv_release_blocks", "kv_truncate", "evict_keys",
           "evict_select_workspace_size", "evict_select", "kva_diag_occupy", "kv_pool_set_threshold",
           "kv_pool_set_active_blocks", "kv_manager_step_workspace_size", "kv_manager_step", "kv_manager_step_select",
           "kva_prefix_index_create", "kva_prefix_index_destroy", "kva_prefix_insert", "kva_prefix_lookup",
           "kva_prefix_remove", "kva_prefix_size", "kva_group_batch", "kva_group_batch_nested",
           "kva_set_option", "kva_get_option"]
PHASE_TILE, PHASE_DECODE, PHASE_MERGE, PHASE_ALL = 1, 2, 4, 7

_lib = None


def lib_path():
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libkvattn.so (building it with nvcc first if missing/stale)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_missing and _build.stale():
        _build.build()
    if not os.path.exists(_build.LIB):
        raise ImportError(f"libkvattn.so not built ({_build.LIB}); run __graft_entry__.build()")
    L = ctypes.CDLL(_build.LIB)
    P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sig = {
        "kva_last_error": ([], ctypes.c_char_p),
        "kva_version": ([], ctypes.c_char_p),
        "kva_validate_batch": ([P, i32, i32], ctypes.c_int),
        "kv_pool_create": ([P, P], ctypes.c_int),
        "kv_pool_destroy": ([P], ctypes.c_int),
        "kv_pool_free_count": ([P, P], ctypes.c_int),
        "kv_pool_resync": ([P], ctypes.c_int),
        "kv_pool_sync": ([P, P], ctypes.c_int),
        "kv_append_workspace_size": ([P, P], ctypes.c_int),
        "kv_append": ([P, P, P, P, i64, P, P, sz, P], ctypes.c_int),
        "hybrid_attention_workspace_size": ([P, P], ctypes.c_int),
        "hybrid_attention_plan": ([P, P, P, sz, P, P], ctypes.c_int),
        "hybrid_attention_run": ([P, P, i64, i64, P, i64, i64, i32, P, P], ctypes.c_int),
        "kv_append_plan": ([P, P, P, P, i64, P, P, sz, P, sz, P, P], ctypes.c_int),
        "hybrid_attention_run_phases": ([P, P, i64, i64, P, i64, i64, i32, P, i32, P], ctypes.c_int),
        "kva_plan_launch_count": ([P, i32, P], ctypes.c_int),
        "kva_plan_set_timing_events": ([P, P, P, P, P], ctypes.c_int),
        "kva_plan_set_span_buffer": ([P, P], ctypes.c_int),
        "kva_plan_set_outputs": ([P, i32, P], ctypes.c_int),
        "kv_release_blocks": ([P, P, i64, P], ctypes.c_int),
        "kv_truncate": ([P, P, P, P], ctypes.c_int),
        "kva_plan_destroy": ([P], ctypes.c_int),
        "kva_plan_get_stats": ([P, P], ctypes.c_int),
        "hybrid_attention": ([P, P, P, i64, i64, P, i64, i64, i32, P, P, sz, P], ctypes.c_int),
        "evict_keys": ([P, P, P, P, i64, P, P], ctypes.c_int),
        "evict_select_workspace_size": ([i64, i64, P], ctypes.c_int),
        "evict_select": ([P, i64, i64, P, P, i32, P, P, sz, P], ctypes.c_int),
        "kva_diag_occupy": ([i32, i32, i64, P], ctypes.c_int),
        "kv_pool_set_threshold": ([P, i64], ctypes.c_int),
        "kv_pool_set_active_blocks": ([P, i64], ctypes.c_int),
        "kv_manager_step_workspace_size": ([P, P, P], ctypes.c_int),
        "kv_manager_step": ([P, P, P, P, P, sz, P], ctypes.c_int),
        "kv_manager_step_select": ([P, P, P, P, P, sz, i64, P, P, sz, P], ctypes.c_int),
        "kva_prefix_index_create": ([P], ctypes.c_int),
        "kva_prefix_index_destroy": ([P], ctypes.c_int),
        "kva_prefix_insert": ([P, P, i64, P, ctypes.c_uint32], ctypes.c_int),
        "kva_prefix_lookup": ([P, P, i64, P, i64, P, ctypes.c_uint32], ctypes.c_int),
        "kva_prefix_remove": ([P, P, i64], ctypes.c_int),
        "kva_prefix_size": ([P, P], ctypes.c_int),
        "kva_group_batch": ([P, i32, P, P, P, i32, P, P, P], ctypes.c_int),
        "kva_group_batch_nested": ([P, i32, P, P, P, i32, P, P, P, P, P], ctypes.c_int),
        "kva_set_option": ([ctypes.c_char_p, i64], ctypes.c_int),
        "kva_get_option": ([ctypes.c_char_p, P], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(st, **extra):
    if st != OK:
        raise KvaError(st, load().kva_last_error().decode(), **extra)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def version() -> str:
    return load().kva_version().decode()


class Pool:
    """kv_pool_create / kv_pool_destroy around caller-owned torch tensors."""

    def __init__(self, k_pool: torch.Tensor, v_pool: torch.Tensor, free_bits: torch.Tensor):
        L = load()
        if not (k_pool.is_cuda and v_pool.is_cuda and free_bits.is_cuda):
            raise KvaError(ERR_INVALID, "pool tensors must be CUDA tensors (no CPU path)")
        assert k_pool.dtype == torch.bfloat16 and k_pool.is_contiguous() and v_pool.is_contiguous()
        nb, hkv, bs, d = k_pool.shape
        self.k_pool, self.v_pool, self.free_bits = k_pool, v_pool, free_bits
        self.desc = PoolDesc(nb, bs, hkv, d, k_pool.data_ptr(), v_pool.data_ptr(),
                             free_bits.data_ptr(), k_pool.device.index or 0)
        self.handle = ctypes.c_void_p()
        _check(L.kv_pool_create(ctypes.byref(self.desc), ctypes.byref(self.handle)))

    def free_count(self) -> int:
        n = ctypes.c_int64()
        _check(load().kv_pool_free_count(self.handle, ctypes.byref(n)))
        return n.value

    def resync(self):
        _check(load().kv_pool_resync(self.handle))

    def sync(self, stream=None):
        """kv_pool_sync (a no-op: every kv_append write is on the caller's stream)."""
        _check(load().kv_pool_sync(self.handle, _stream(stream)))

    def set_threshold(self, threshold_blocks: int):
        """kv_pool_set_threshold: burst reserve for kv_append (< 0 disables)."""
        _check(load().kv_pool_set_threshold(self.handle, int(threshold_blocks)))

    def set_active_blocks(self, n: int):
        """kv_pool_set_active_blocks: active-class block count (e.g. the manager step's)."""
        _check(load().kv_pool_set_active_blocks(self.handle, int(n)))

    def close(self):
        if self.handle:
            load().kv_pool_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch:
    """The batch descriptor (host numpy arrays + the device block table)."""

    def __init__(self, batch: dict, device):
        self.q_indptr = np.ascontiguousarray(batch["q_indptr"], np.int32)
        self.ctx_len = np.ascontiguousarray(batch["ctx_len"], np.int32)
        self.req_type = np.ascontiguousarray(batch.get("req_type", np.zeros(len(self.ctx_len))), np.int32)
        self.table_host = np.ascontiguousarray(batch["block_table"], np.int32).copy()
        self.group_of = (None if batch.get("group_of") is None
                         else np.ascontiguousarray(batch["group_of"], np.int32))
        gpb = batch.get("group_prefix_blocks")
        self.group_prefix_blocks = np.ascontiguousarray(gpb if gpb is not None else [], np.int32)
        gpa = batch.get("group_parent")
        self.group_parent = None if gpa is None else np.ascontiguousarray(gpa, np.int32)
        self.table_dev = (torch.from_numpy(self.table_host.copy()).to(device)
                          if device is not None else torch.from_numpy(self.table_host.copy()))
        self.num_reqs = len(self.ctx_len)
        self.num_q_heads = int(batch["num_q_heads"])
        self.num_kv_heads = int(batch["num_kv_heads"])
        self.head_dim = int(batch["head_dim"])
        self.sm_scale = float(batch.get("sm_scale", 0.0) or 0.0)
        self.total_q = int(self.q_indptr[-1]) if len(self.q_indptr) else 0
        self._desc = None

    def __setattr__(self, name, value):
        # any rebinding (a new array / tensor object) invalidates the cached descriptor; in-place
        # writes into the arrays keep their addresses and need no rebuild
        if name != "_desc":
            object.__setattr__(self, "_desc", None)
        object.__setattr__(self, name, value)

    def desc(self):
        """The C descriptor (cached: building it costs ~8 us of ctypes marshalling per call)."""
        d = self._desc
        if d is not None and d.block_table == self.table_dev.data_ptr():
            return d
        a = lambda x: None if x is None else x.ctypes.data
        d = BatchDesc(self.num_reqs, self.num_q_heads, self.num_kv_heads, self.head_dim,
                      a(self.req_type), a(self.q_indptr), a(self.ctx_len), self.table_dev.data_ptr(),
                      a(self.table_host), self.table_host.shape[1], a(self.group_of),
                      len(self.group_prefix_blocks), a(self.group_prefix_blocks) if len(self.group_prefix_blocks) else None,
                      self.sm_scale, a(self.group_parent) if self.group_parent is not None and len(self.group_parent) else None)
        self._desc = d  # keep alive
        return d

    def as_dict(self):
        """Descriptor as a dict of host arrays (for the oracle in tests)."""
        return dict(num_reqs=self.num_reqs, num_q_heads=self.num_q_heads,
                    num_kv_heads=self.num_kv_heads, head_dim=self.head_dim,
                    q_indptr=self.q_indptr, ctx_len=self.ctx_len, block_table=self.table_host,
                    group_of=self.group_of, group_prefix_blocks=self.group_prefix_blocks,
                    sm_scale=self.sm_scale)


def validate_batch(batch: "Batch", num_blocks: int, mode: int = 0) -> int:
    """Host-only descriptor check; returns the status code (0 = OK)."""
    return load().kva_validate_batch(ctypes.byref(batch.desc()), num_blocks, mode)


def last_error() -> str:
    return load().kva_last_error().decode()


def _workspace(nbytes, device, stream=None):
    """Default scratch for a call enqueued on `stream`.  The caching allocator tracks the
    stream a block was allocated on; the block is marked as used by `stream` as well, so it is
    not handed to a new allocation before `stream`'s work on it has finished."""
    ws = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
    if stream is not None and stream != torch.cuda.current_stream(ws.device):
        ws.record_stream(stream)
    return ws


def kv_append_workspace_size(batch: Batch) -> int:
    n = ctypes.c_size_t()
    _check(load().kv_append_workspace_size(ctypes.byref(batch.desc()), ctypes.byref(n)))
    return n.value


def kv_append(pool: Pool, batch: Batch, k_new: torch.Tensor, v_new: torch.Tensor,
              workspace: torch.Tensor | None = None, stream=None):
    """Append K/V rows [total_q][Hkv][d] (a2).  Raises KvaError(NEEDS_EVICTION, deficit=...)."""
    L = load()
    d = batch.desc()
    if workspace is None:
        workspace = _workspace(kv_append_workspace_size(batch), k_new.device, stream)
    deficit = ctypes.c_int32(0)
    st = L.kv_append(pool.handle, ctypes.byref(d), _ptr(k_new), _ptr(v_new), k_new.stride(0),
                     ctypes.byref(deficit), _ptr(workspace), workspace.numel(), _stream(stream))
    _check(st, deficit=deficit.value)
    return workspace


def kv_append_plan(pool: Pool, batch: Batch, k_new: torch.Tensor, v_new: torch.Tensor,
                   append_workspace: torch.Tensor | None = None, attn_workspace: torch.Tensor | None = None,
                   stream=None) -> "Plan":
    """kv_append + hybrid_attention_plan of the same descriptor in one library call (one
    validation); returns the Plan.  Raises KvaError(NEEDS_EVICTION, deficit=...)."""
    if append_workspace is None:
        append_workspace = _workspace(kv_append_workspace_size(batch), k_new.device, stream)
    if attn_workspace is None:
        attn_workspace = _workspace(hybrid_attention_workspace_size(batch), k_new.device, stream)
    deficit = ctypes.c_int32(0)
    h = ctypes.c_void_p()
    st = load().kv_append_plan(pool.handle, ctypes.byref(batch.desc()), _ptr(k_new), _ptr(v_new), k_new.stride(0),
                               ctypes.byref(deficit), _ptr(append_workspace), append_workspace.numel(),
                               _ptr(attn_workspace), attn_workspace.numel(), _stream(stream), ctypes.byref(h))
    _check(st, deficit=deficit.value)
    plan = Plan(pool, batch, attn_workspace, _handle=h)
    plan.append_workspace = append_workspace
    return plan


def hybrid_attention_workspace_size(batch: Batch) -> int:
    n = ctypes.c_size_t()
    _check(load().hybrid_attention_workspace_size(ctypes.byref(batch.desc()), ctypes.byref(n)))
    return n.value


class Plan:
    """hybrid_attention_plan: work lists uploaded into `workspace`; reusable by run()."""

    def __init__(self, pool: Pool, batch: Batch, workspace: torch.Tensor | None = None, stream=None,
                 device=None, _handle=None):
        device = device or pool.k_pool.device
        if workspace is None:
            workspace = _workspace(hybrid_attention_workspace_size(batch), device, stream)
        self.workspace = workspace
        self.pool = pool  # the C plan uses the pool's side stream / events: keep it alive
        self.batch = batch
        if _handle is not None:  # made by kv_append_plan
            self.handle = _handle
            return
        self.handle = ctypes.c_void_p()
        _check(load().hybrid_attention_plan(pool.handle, ctypes.byref(batch.desc()), _ptr(workspace),
                                            workspace.numel(), _stream(stream), ctypes.byref(self.handle)))

    def stats(self) -> dict:
        s = PlanStats()
        _check(load().kva_plan_get_stats(self.handle, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in PlanStats._fields_}

    def run(self, q: torch.Tensor, out: torch.Tensor, lse: torch.Tensor | None = None, stream=None,
            phases: int = PHASE_ALL):
        out_dtype = OUT_F32 if out.dtype == torch.float32 else OUT_BF16
        if out.dtype not in (torch.float32, torch.bfloat16):
            raise KvaError(ERR_INVALID, "out must be bf16 or fp32")
        _check(load().hybrid_attention_run_phases(self.handle, _ptr(q), q.stride(0), q.stride(1),
                                                  _ptr(out), out.stride(0), out.stride(1), out_dtype,
                                                  _ptr(lse), phases, _stream(stream)))
        return out

    def set_timing_events(self, tile_begin=None, tile_end=None, decode_begin=None, decode_end=None):
        """torch.cuda.Event objects (already recorded once, so their handles exist)."""
        h = lambda e: None if e is None else ctypes.c_void_p(e.cuda_event)
        _check(load().kva_plan_set_timing_events(self.handle, h(tile_begin), h(tile_end),
                                                 h(decode_begin), h(decode_end)))

    def set_extra_outputs(self, outs):
        """kva_plan_set_outputs: every output row is also stored into each of `outs` (device
        tensors or raw device addresses with out's strides) — the fused all-gather epilogue."""
        ptrs = [o if isinstance(o, int) else o.data_ptr() for o in (outs or [])]
        self._extra_refs = list(outs or [])  # keep tensors alive while the plan may run
        arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
        _check(load().kva_plan_set_outputs(self.handle, len(ptrs), arr))

    def set_span_buffer(self, span: torch.Tensor | None):
        """kva_plan_set_span_buffer: int64 device tensor [6] (decode, tile, merge start/end ns;
        initialise [0], [2], [4] to -1 (= UINT64_MAX bits) and [1], [3], [5] to 0)."""
        if span is not None and span.numel() < 6:
            raise KvaError(ERR_INVALID, "span buffer needs 6 entries")
        _check(load().kva_plan_set_span_buffer(self.handle, _ptr(span) if span is not None else None))

    def launch_count(self, phases: int = PHASE_ALL) -> int:
        n = ctypes.c_int32()
        _check(load().kva_plan_launch_count(self.handle, phases, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.handle:
            load().kva_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hybrid_attention(pool: Pool, batch: Batch, q: torch.Tensor, out: torch.Tensor | None = None,
                     lse: torch.Tensor | None = None, out_dtype=torch.bfloat16,
                     workspace: torch.Tensor | None = None, stream=None):
    """One attention step of the mixed batch (plan + run).  q: [total_q][Hq][d] bf16."""
    L = load()
    if out is None:
        out = torch.empty(q.shape, dtype=out_dtype, device=q.device)
    if workspace is None:
        workspace = _workspace(hybrid_attention_workspace_size(batch), q.device, stream)
    od = OUT_F32 if out.dtype == torch.float32 else OUT_BF16
    _check(L.hybrid_attention(pool.handle, ctypes.byref(batch.desc()), _ptr(q), q.stride(0),
                              q.stride(1), _ptr(out), out.stride(0), out.stride(1), od, _ptr(lse),
                              _ptr(workspace), workspace.numel(), _stream(stream)))
    return out


def kv_truncate(pool: Pool, batch: Batch, keep_len, stream=None):
    """Shorten request i to its first keep_len[i] tokens (-1: untouched): its blocks past that
    are released and their table entries reset to -1 (host mirror and device table)."""
    a = np.ascontiguousarray(keep_len, np.int32)
    if a.size != batch.num_reqs:
        raise KvaError(ERR_INVALID, "keep_len must have num_reqs entries")
    _check(load().kv_truncate(pool.handle, ctypes.byref(batch.desc()), a.ctypes.data, _stream(stream)))


def kv_release_blocks(pool: Pool, ids, stream=None):
    """Return blocks (host int32 ids) to the free pool (recompute-mode release)."""
    a = np.ascontiguousarray(ids, np.int32)
    _check(load().kv_release_blocks(pool.handle, a.ctypes.data if a.size else None, a.size,
                                    _stream(stream)))


def evict_keys(state, rc, lat, depth=None, keys=None, stream=None):
    """priority_of as u64 keys (a8) on device tensors (uint8/int32-as-u32/int16-as-u16)."""
    L = load()
    n = state.numel()
    if keys is None:
        keys = torch.empty(n, dtype=torch.int64, device=state.device)
    _check(L.evict_keys(_ptr(state), _ptr(rc), _ptr(lat), _ptr(depth), n, _ptr(keys), _stream(stream)))
    return keys


class ManagerStep:
    """kv_manager_step: class transitions (host chains, list order, last wins),
    rc recount from the offline pool's chains (device ids), active-class count, eviction keys.
    The host arrays are marshalled once per call; every step of the pass runs in the library."""

    def __init__(self, state, rc, lat, depth=None):
        self.state, self.rc, self.lat, self.depth = state, rc, lat, depth
        self.meta = BlockMeta(state.numel(), _ptr(state), _ptr(rc), _ptr(lat), _ptr(depth))
        self.keys = torch.empty(state.numel(), dtype=torch.int64, device=state.device)
        self.n_active = torch.zeros(1, dtype=torch.int64, device=state.device)
        self.ws = torch.empty(256, dtype=torch.uint8, device=state.device)

    @staticmethod
    def chains_to_device(csr, device):
        """A chains_csr() tuple as device tensors (kva_manager_update.chains_on_device): the
        call then uploads nothing and the ids are range-checked on the device."""
        ci, cids, cst = csr
        return (torch.from_numpy(np.ascontiguousarray(ci, np.int32)).to(device),
                torch.from_numpy(np.ascontiguousarray(cids[: int(ci[-1])], np.int32)).to(device),
                torch.from_numpy(np.ascontiguousarray(cst, np.uint8)).to(device))

    @staticmethod
    def chains_csr(chains):
        """[(state, ids-array), ...] -> host CSR (indptr, ids, states) for __call__."""
        ci = np.zeros(len(chains) + 1, np.int32)
        for j, (_, ids) in enumerate(chains):
            ci[j + 1] = ci[j] + len(ids)
        cids = (np.concatenate([np.asarray(ids, np.int32) for _, ids in chains]) if chains
                else np.zeros(1, np.int32))
        cst = np.array([s_ for s_, _ in chains] or [0], np.uint8)
        return ci, cids, cst

    def __call__(self, now: int, chains, pool_ids: torch.Tensor | None, del_ids: torch.Tensor | None = None,
                 recount: bool = True, stream=None, select=None):
        """chains: [(state, ids-array), ...] or a chains_csr() tuple (host); pool_ids: device
        int32 (recount: every pool chain; incremental: the chains that joined), del_ids: device
        int32 (incremental: the chains that left).  select = (k, out_ids, sel_workspace): the
        eviction order of the new keys in the same kernel (kv_manager_step_select; the count
        stays on the device in sel_workspace[:8])."""
        ci, cids, cst = chains if isinstance(chains, tuple) else self.chains_csr(chains)
        plen = pool_ids.numel() if pool_ids is not None else 0
        dlen = del_ids.numel() if del_ids is not None else 0
        on_dev = isinstance(ci, torch.Tensor)  # device CSR (chains_to_device): no upload
        L = load()
        # the marshalled update is reused while the same arrays / tensors are passed (the cache
        # holds references, so an identity cannot be recycled while cached); in-place edits of
        # the arrays keep their addresses
        n_ids = (int(cids.numel()) if on_dev else (int(ci[-1]) if len(ci) else 0))
        key = (ci, cids, cst, pool_ids, del_ids, plen, dlen, n_ids)
        c = getattr(self, "_ucache", None)
        if (c is None or any(a is not b for a, b in zip(c[0][:5], key[:5])) or c[0][5:] != key[5:]):
            ptr = _ptr if on_dev else (lambda a: a.ctypes.data)
            nch = (ci.numel() if on_dev else len(ci)) - 1
            u = ManagerUpdate(0, nch, ptr(ci), ptr(cids), ptr(cst), 0,
                              _ptr(pool_ids) if plen else None, plen, _ptr(del_ids) if dlen else None, dlen,
                              1 if on_dev else 0, n_ids)
            need = ctypes.c_size_t()
            _check(L.kv_manager_step_workspace_size(ctypes.byref(self.meta), ctypes.byref(u), ctypes.byref(need)))
            c = self._ucache = (key, u, need.value)
        _, u, need_b = c
        u.now = int(now) & 0xFFFFFFFF
        u.recount = 1 if recount else 0
        if self.ws.numel() < need_b:
            self.ws = torch.empty(need_b, dtype=torch.uint8, device=self.state.device)
        if select is None:
            _check(L.kv_manager_step(ctypes.byref(self.meta), ctypes.byref(u), _ptr(self.keys), _ptr(self.n_active),
                                     _ptr(self.ws), self.ws.numel(), _stream(stream)))
            return self.keys
        k, out_ids, sel_ws = select
        _check(L.kv_manager_step_select(ctypes.byref(self.meta), ctypes.byref(u), _ptr(self.keys),
                                        _ptr(self.n_active), _ptr(self.ws), self.ws.numel(), int(k), _ptr(out_ids),
                                        _ptr(sel_ws), sel_ws.numel(), _stream(stream)))
        return self.keys


def evict_select_workspace_size(n: int, k: int) -> int:
    b = ctypes.c_size_t()
    _check(load().evict_select_workspace_size(n, k, ctypes.byref(b)))
    return b.value


def evict_select(keys: torch.Tensor, k: int, out_ids: torch.Tensor | None = None, apply: bool = False,
                 pool: Pool | None = None, workspace: torch.Tensor | None = None, stream=None,
                 allow_short: bool = True, sync: bool = True):
    """The k blocks with the smallest (key, id), in eviction order.  Returns (ids, n_selected);
    with sync=False nothing waits for the device and n_selected is None."""
    L = load()
    n = keys.numel()
    if out_ids is None:
        out_ids = torch.empty(max(k, 1), dtype=torch.int32, device=keys.device)
    if workspace is None:
        workspace = _workspace(evict_select_workspace_size(n, k), keys.device, stream)
    nsel = ctypes.c_int64(0)
    if not sync:
        _check(L.evict_select(_ptr(keys), n, k, _ptr(out_ids), None, int(bool(apply)),
                              pool.handle if pool is not None else None, _ptr(workspace),
                              workspace.numel(), _stream(stream)))
        return out_ids, None
    st = L.evict_select(_ptr(keys), n, k, _ptr(out_ids), ctypes.byref(nsel), int(bool(apply)),
                        pool.handle if pool is not None else None, _ptr(workspace), workspace.numel(),
                        _stream(stream))
    if st == EVICTION_SHORT and allow_short:
        return out_ids[: nsel.value], nsel.value
    _check(st)
    return out_ids[: nsel.value], nsel.value


def set_option(name: str, value: int):
    """kva_set_option (include/kvattn.h): process-wide tuning / diagnostics option."""
    _check(load().kva_set_option(name.encode(), int(value)))


def get_option(name: str) -> int:
    v = ctypes.c_int64()
    _check(load().kva_get_option(name.encode(), ctypes.byref(v)))
    return v.value


class options:
    """Context manager: `with options(tile_ctas=40, overlap=1): ...` restores the old values."""

    def __init__(self, **kw):
        self.kw, self.old = kw, {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)


def free_bits_tensor(free_bits_np: np.ndarray, device) -> torch.Tensor:
    """uint32 numpy bitmap -> int32 device tensor with the same bits."""
    return torch.from_numpy(np.ascontiguousarray(free_bits_np, np.uint32).view(np.int32).copy()).to(device)


def diag_occupy(n_ctas: int, smem_bytes: int, ns: int, stream=None):
    """Diagnostics: hold n_ctas SMs (smem_bytes each) for ns nanoseconds on `stream`."""
    _check(load().kva_diag_occupy(n_ctas, smem_bytes, ns, _stream(stream)))


class PrefixIndex:
    """Block-granular prefix index (host, C++): insert / lookup / remove chains of
    whole 16-token blocks and build the batch descriptor's shared-prefix groups (group_batch)."""

    def __init__(self):
        self.handle = ctypes.c_void_p()
        _check(load().kva_prefix_index_create(ctypes.byref(self.handle)))

    @staticmethod
    def _i32(a):
        return np.ascontiguousarray(a, dtype=np.int32)

    def insert(self, tokens, block_ids, now: int = 0):
        t, b = self._i32(tokens), self._i32(block_ids)
        _check(load().kva_prefix_insert(self.handle, t.ctypes.data, t.size, b.ctypes.data, int(now) & 0xFFFFFFFF))

    def lookup(self, tokens, now: int = 0) -> np.ndarray:
        t = self._i32(tokens)
        out = np.zeros(max(1, t.size // 16), np.int32)
        n = ctypes.c_int64()
        _check(load().kva_prefix_lookup(self.handle, t.ctypes.data, t.size, out.ctypes.data, out.size,
                                        ctypes.byref(n), int(now) & 0xFFFFFFFF))
        return out[: n.value]

    def remove(self, block_ids):
        b = self._i32(block_ids)
        _check(load().kva_prefix_remove(self.handle, b.ctypes.data, b.size))

    def size(self) -> int:
        n = ctypes.c_int64()
        _check(load().kva_prefix_size(self.handle, ctypes.byref(n)))
        return n.value

    def group_batch(self, token_lists, prefix_limit_blocks=None, min_blocks: int = 1):
        """-> (group_of int32[R], group_prefix_blocks int32[G]) for the batch descriptor."""
        arrs = [self._i32(t) for t in token_lists]
        R = len(arrs)
        ptrs = (ctypes.c_void_p * max(1, R))(*[a.ctypes.data for a in arrs])
        lens = np.array([a.size for a in arrs] or [0], np.int64)
        lim = None if prefix_limit_blocks is None else self._i32(prefix_limit_blocks)
        gof = np.full(max(1, R), -1, np.int32)
        gpb = np.zeros(max(1, R), np.int32)
        G = ctypes.c_int32()
        _check(load().kva_group_batch(self.handle, R, ptrs, lens.ctypes.data,
                                      None if lim is None else lim.ctypes.data, int(min_blocks),
                                      gof.ctypes.data, gpb.ctypes.data, ctypes.byref(G)))
        return gof[:R], gpb[: G.value]

    def group_batch_nested(self, token_lists, level_min_blocks, prefix_limit_blocks=None):
        """-> (group_of[R], group_prefix_blocks[G], group_parent[G]) for nested groups."""
        arrs = [self._i32(t) for t in token_lists]
        R = len(arrs)
        ptrs = (ctypes.c_void_p * max(1, R))(*[a.ctypes.data for a in arrs])
        lens = np.array([a.size for a in arrs] or [0], np.int64)
        lim = None if prefix_limit_blocks is None else self._i32(prefix_limit_blocks)
        lv = self._i32(level_min_blocks)
        gof = np.full(max(1, R), -1, np.int32)
        gpb = np.zeros(max(1, R), np.int32)
        gpa = np.zeros(max(1, R), np.int32)
        G = ctypes.c_int32()
        _check(load().kva_group_batch_nested(self.handle, R, ptrs, lens.ctypes.data,
                                             None if lim is None else lim.ctypes.data, lv.size, lv.ctypes.data,
                                             gof.ctypes.data, gpb.ctypes.data, gpa.ctypes.data, ctypes.byref(G)))
        return gof[:R], gpb[: G.value], gpa[: G.value]

    def close(self):
        if self.handle:
            load().kva_prefix_index_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
