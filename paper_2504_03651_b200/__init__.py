"""B200-native hybrid paged attention for co-scheduled online/offline LLM serving
(arxiv 2504.03651 hot path): C-ABI library libkvattn.so + thin ctypes binding.

The product path is the CUDA library only; importing this package does not touch the
oracle (oracle/ is test infrastructure).
"""
from .kvattn import (  # noqa: F401
    Batch, KvaError, Plan, Pool, evict_keys, evict_select, evict_select_workspace_size,
    free_bits_tensor, hybrid_attention, hybrid_attention_workspace_size, kv_append, kv_release_blocks, kv_truncate,
    PHASE_TILE, PHASE_DECODE, PHASE_MERGE, PHASE_ALL,
    kv_append_workspace_size, kv_append_plan, last_error, load, validate_batch, version,
    OK, ERR_INVALID, ERR_UNSUPPORTED, NEEDS_EVICTION, ERR_CAPACITY, EVICTION_SHORT, ERR_GROUP,
    ERR_CUDA, OUT_BF16, OUT_F32, diag_occupy, ManagerStep, PrefixIndex, set_option, get_option, options,
)
