/*
 * kvattn.h — C ABI of the B200-native hybrid paged-attention library (libkvattn.so).
 *
 * The library implements the device hot path of one iteration of the co-scheduled
 * online/offline serving loop of arxiv 2504.03651 (citation keys: P:n = PAPER.md line n,
 * S:n = SPEC.md line n; "reading #n" = DESIGN.md §3):
 *   1. kv_append        — append this iteration's K/V into the paged pool, allocating
 *                          blocks deterministically ("appending the corresponding KV
 *                          state to the cache"; P:328 fixed-size blocks; Eq.(5)).
 *   2. hybrid_attention — one attention step for a MIXED batch of online decodes and
 *                          offline chunked prefills in which
 *                          offline tasks share resident prefix blocks.
 *   3. evict_keys/evict_select — the task-aware eviction order: priority then
 *                          last access time, as kept by the free table.
 *
 * Conventions (all calls):
 *   - Every call returns kva_status; nothing throws or exits across the ABI.  On error a
 *     thread-local message is available from kva_last_error().
 *   - All descriptor validation runs on the host, synchronously, BEFORE anything is
 *     enqueued; an error status means no device work was enqueued and no state changed.
 *   - Device work is enqueued on the caller's stream (NULL = legacy default stream) and
 *     the call returns after enqueue, except where a host output needs a device result
 *     (documented per call: evict_select's n_selected, kv_pool_create's free count).
 *   - Pointers marked "device" must be device memory of the pool's device; "host" are host
 *     memory.  All device buffers are caller-owned (PyTorch allocates them); the library
 *     owns only its opaque handles, host planning scratch and pinned staging buffers.
 *   - bf16 = IEEE bfloat16 bit pattern (uint16).  Block size is fixed at 16 tokens
 *     (reading #5).  head_dim must be 64 or 128 (else KVA_ERR_UNSUPPORTED).
 *   - Single writer per pool: calls on one pool (kv_append, kv_append_plan,
 *     hybrid_attention_plan / _run, kv_release_blocks, kv_truncate, evict_select with apply,
 *     kv_pool_*) must be serialised by the caller, and so must the runs of one plan; the library
 *     does not lock them (it only guards its upload staging ring).
 *   - *_workspace_size calls validate the descriptor exactly as the call they size does (minus
 *     the block-id range, which needs the pool) and return that status on error.
 */
#ifndef KVATTN_H_
#define KVATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *kva_stream_t; /* == cudaStream_t */

typedef enum {
  KVA_OK = 0,
  KVA_ERR_INVALID = 1,      /* shape / pointer / descriptor error ("domain error") */
  KVA_ERR_UNSUPPORTED = 2,  /* head_dim not in {64,128}, block_size != 16, ...            */
  KVA_NEEDS_EVICTION = 3,   /* kv_append: free blocks < needed; *deficit_blocks set;
                               NO state change                                 */
  KVA_ERR_CAPACITY = 4,     /* one request needs more blocks than the pool has      */
  KVA_EVICTION_SHORT = 5,   /* evict_select: fewer than k evictable blocks; the first
                               n_selected ids are valid (S:147 EvictionImpossible)         */
  KVA_ERR_GROUP = 6,        /* shared-prefix precondition violated (reading #8)             */
  KVA_ERR_CUDA = 7          /* CUDA runtime / launch error                                  */
} kva_status;

/* Thread-local text of the last error (never NULL). */
const char *kva_last_error(void);
/* Library build string (compile target, version). */
const char *kva_version(void);

/* ------------------------------------------------------------------------------------
 * Pool.  The paged KV cache of P:328 ("the KV cache is divided into fixed-sized blocks
 * ... enabling efficient and non-contiguous memory allocation").
 *   k_pool, v_pool : device bf16 [num_blocks][num_kv_heads][16][head_dim]  (caller-owned)
 *                    num_kv_heads is the LOCAL count (heads sharded over G ranks, §8(e)).
 *   free_bits      : device uint32 [ceil(num_blocks/32)], bit b%32 of word b/32 set = block
 *                    b free (caller-owned).  The library keeps a host mirror of it (it is
 *                    the single writer after create) and uses it to allocate blocks.
 * kv_pool_create reads free_bits once (synchronous device->host copy).
 * ------------------------------------------------------------------------------------ */
typedef struct kva_pool kva_pool;
typedef struct {
  int32_t num_blocks;
  int32_t block_size;   /* must be 16 */
  int32_t num_kv_heads; /* local */
  int32_t head_dim;     /* 64 | 128 */
  void *k_pool;
  void *v_pool;
  uint32_t *free_bits;
  int32_t device;       /* CUDA ordinal the buffers live on */
} kva_pool_desc;

kva_status kv_pool_create(const kva_pool_desc *desc, kva_pool **out);
/* Frees library-owned host state only; never frees caller memory. */
kva_status kv_pool_destroy(kva_pool *pool);
/* Number of free blocks according to the library's mirror (host, no sync). */
kva_status kv_pool_free_count(const kva_pool *pool, int64_t *n_free);
/* Re-read free_bits from the device (synchronous) after the caller edited it. */
kva_status kv_pool_resync(kva_pool *pool);
/* No-op (every kv_append write is on the caller's stream; see kv_append "Ordering"). */
kva_status kv_pool_sync(kva_pool *pool, kva_stream_t stream);

/* ------------------------------------------------------------------------------------
 * Batch descriptor: the iteration's batch T_i of prefill chunks + decode tokens (P:172,
 * P:226-228).  R = num_reqs.  Request i owns query rows [q_indptr[i], q_indptr[i+1])
 * (q_len_i = q_indptr[i+1]-q_indptr[i] >= 1) at absolute positions [ctx_i - q_len_i, ctx_i);
 * ctx_len[i] is its KV length AFTER this step's append (readings #2-#4).  A query at
 * position p attends to keys [0, p] (causal).
 * Shared-prefix groups: group_of[i] = -1 or a group index;
 * group g covers the first group_prefix_blocks[g] blocks; every member's first
 * group_prefix_blocks[g] table entries must equal the group's blocks (those of its first
 * member) and every member's queries must lie after the prefix, else KVA_ERR_GROUP.
 * Grouping never changes results (reading #7); it changes how blocks are read.
 * Nested groups (multi-level cascade; e.g. a system prompt shared by every
 * offline task and a document shared by a subset): group_parent[g] = -1 or a group p < g with
 * group_prefix_blocks[p] <= group_prefix_blocks[g] whose blocks are the first
 * group_prefix_blocks[p] blocks of g; a request names its DEEPEST group.  Decode-class members
 * then read each level's blocks once per (level, kv head), stacked over every member below it
 * (at most KVA_MAX_CASCADE = 4 levels).  group_parent = NULL: every group is a root.
 * ------------------------------------------------------------------------------------ */
enum { KVA_MAX_CASCADE = 4 };
enum { KVA_ONLINE_DECODE = 0, KVA_OFFLINE_PREFILL = 1, KVA_OFFLINE_DECODE = 2,
       KVA_ONLINE_PREFILL = 3 };
enum { KVA_OUT_BF16 = 0, KVA_OUT_F32 = 1 };

typedef struct {
  int32_t num_reqs;
  int32_t num_q_heads;              /* local; num_q_heads % num_kv_heads == 0 */
  int32_t num_kv_heads;             /* local; must equal the pool's */
  int32_t head_dim;
  const int32_t *req_type;          /* host [R]; planning/metrics only (nullable) */
  const int32_t *q_indptr;          /* host [R+1], q_indptr[0] = 0, non-decreasing */
  const int32_t *ctx_len;           /* host [R] */
  int32_t *block_table;             /* device [R][max_blocks] int32, -1 = unallocated */
  int32_t *block_table_host;        /* host mirror [R][max_blocks]; kv_append writes the
                                       ids it allocates into BOTH tables */
  int32_t max_blocks;
  const int32_t *group_of;          /* host [R] (nullable = no groups) */
  int32_t num_groups;
  const int32_t *group_prefix_blocks; /* host [num_groups] */
  float sm_scale;                   /* <= 0 -> 1/sqrt(head_dim) (reading #1) */
  const int32_t *group_parent;      /* host [num_groups], -1 = root (nullable = all roots) */
} kva_batch_desc;

/* Host-only descriptor check (no device work): mode 0 = as hybrid_attention validates it
 * (every block of [0, ctx) allocated), mode 1 = as kv_append does (resident part only).
 * Returns the status the corresponding call would return for descriptor errors. */
kva_status kva_validate_batch(const kva_batch_desc *desc, int32_t num_blocks, int32_t mode);

/* ------------------------------------------------------------------------------------
 * kv_append (a2).  For each request in descriptor order and each new position t in
 * [ctx-q_len, ctx) ascending: if table[i][t/16] == -1 the smallest free block id is taken
 * (reading #13; a partially filled last block is filled first, reading #14), then the K/V
 * row of every local kv-head is written to slot (table[i][t/16], t % 16).
 *   k_new, v_new : device bf16 [total_q][num_kv_heads][head_dim]; token stride
 *                  new_stride_tok elements (>= num_kv_heads*head_dim), heads contiguous.
 *   workspace    : device scratch of kv_append_workspace_size() bytes (16-B aligned).
 * Ordering: everything is enqueued on `stream` in two kernels: (1) the rows of decode-class
 *   requests (q_len * Hq/Hkv <= 16; their <= 2 blocks resolved on the host) together with the
 *   new table entries and free bits, (2) the rows of the other requests (read only by the
 *   tensor-core tile kernel, which hybrid_attention_run launches with programmatic dependent
 *   launch so that it becomes resident while (2) still writes, and waits for it in-kernel).
 *   kv_pool_sync is a no-op kept for callers written against an earlier side-stream variant.
 * Errors: KVA_NEEDS_EVICTION (needed > free, *deficit_blocks = needed - free, nothing
 * enqueued); KVA_ERR_CAPACITY (ceil(ctx/16) > num_blocks for some request);
 * KVA_ERR_GROUP (an appended position inside a group prefix); KVA_ERR_INVALID.
 * ------------------------------------------------------------------------------------ */
kva_status kv_append_workspace_size(const kva_batch_desc *desc, size_t *bytes);
kva_status kv_append(kva_pool *pool, kva_batch_desc *desc, const void *k_new,
                     const void *v_new, int64_t new_stride_tok, int32_t *deficit_blocks,
                     void *workspace, size_t workspace_bytes, kva_stream_t stream);

/* ------------------------------------------------------------------------------------
 * hybrid_attention (a1 plan + a3..a6).  out[row][h][:] = softmax over keys [0, p] of
 * (q . k) * sm_scale, times V, for every query row and local q-head h (kv-head
 * h / (Hq/Hkv), reading #9); lse[row][h] = natural-log log-sum-exp of the scaled scores.
 *   q   : device bf16, element (row, h, c) at q[row*q_stride_tok + h*q_stride_head + c]
 *   out : device, bf16 (KVA_OUT_BF16) or fp32 (KVA_OUT_F32), same indexing with o_stride_*
 *   lse : device fp32 [total_q][num_q_heads] (nullable)
 *   workspace : device scratch of hybrid_attention_workspace_size() bytes.
 * hybrid_attention = hybrid_attention_plan + hybrid_attention_run.  The plan (host work
 * lists uploaded into the workspace on `stream`) can be reused by several runs — e.g.
 * every layer of a model — while the descriptor is unchanged; runs enqueue kernels only
 * (CUDA-graph capturable).  Errors: KVA_ERR_GROUP, KVA_ERR_INVALID, KVA_ERR_UNSUPPORTED.
 * ------------------------------------------------------------------------------------ */
typedef struct kva_plan kva_plan;
kva_status hybrid_attention_workspace_size(const kva_batch_desc *desc, size_t *bytes);
kva_status hybrid_attention_plan(kva_pool *pool, const kva_batch_desc *desc, void *workspace,
                                 size_t workspace_bytes, kva_stream_t stream, kva_plan **plan);
/* kv_append followed by hybrid_attention_plan of the same descriptor, in one call (the serving
 * iteration's order: append the step's K/V, then attend).  Same arguments, errors
 * and effects as the two calls in sequence; the descriptor is validated once: kv_append checks
 * the resident part and writes every new position's table entry itself, which is what the
 * plan's own check would re-verify.  The plan is made first (it reads no block id), then the
 * append: on ANY error (KVA_NEEDS_EVICTION with *deficit_blocks, a workspace too small, ...)
 * the pool, the tables and the free bitmap are unchanged and no plan is returned (the plan's
 * work lists may already have been uploaded into attn_workspace).  *plan is owned by the
 * caller (kva_plan_destroy). */
kva_status kv_append_plan(kva_pool *pool, kva_batch_desc *desc, const void *k_new, const void *v_new,
                          int64_t new_stride_tok, int32_t *deficit_blocks, void *append_workspace,
                          size_t append_workspace_bytes, void *attn_workspace, size_t attn_workspace_bytes,
                          kva_stream_t stream, kva_plan **plan);
kva_status hybrid_attention_run(const kva_plan *plan, const void *q, int64_t q_stride_tok,
                                int64_t q_stride_head, void *out, int64_t o_stride_tok,
                                int64_t o_stride_head, int32_t out_dtype, float *lse,
                                kva_stream_t stream);
/* Run only some phases of a plan (profiling / per-kernel timing inside a step); phases is a
 * mask of KVA_PHASE_*.  Running TILE|DECODE then MERGE in order equals hybrid_attention_run. */
enum { KVA_PHASE_TILE = 1, KVA_PHASE_DECODE = 2, KVA_PHASE_MERGE = 4, KVA_PHASE_ALL = 7 };
kva_status hybrid_attention_run_phases(const kva_plan *plan, const void *q, int64_t q_stride_tok,
                                       int64_t q_stride_head, void *out, int64_t o_stride_tok,
                                       int64_t o_stride_head, int32_t out_dtype, float *lse,
                                       int32_t phases, kva_stream_t stream);
/* Instrumentation: cudaEvent_t handles (or NULL) recorded immediately before/after the tile
 * kernel launch (on the stream it runs on) and the decode kernel launch (on the caller's
 * stream) by every later run of this plan — per-kernel timing inside an overlapped step. */
/* Instrumentation without stream operations: if dev_span (device, 6 x u64) is set, every later
 * run of this plan records %globaltimer nanoseconds: [0] = min start and [1] = max end over the
 * decode kernel's CTAs, [2] / [3] = the same for the tile kernel, [4] / [5] for the merge kernel
 * (atomicMin / atomicMax: the caller initialises [0], [2], [4] to UINT64_MAX and [1], [3], [5]
 * to 0).  Unlike timing events this does not break the programmatic-dependent-launch chain of
 * the run.  NULL disables it. */
kva_status kva_plan_set_span_buffer(kva_plan *plan, unsigned long long *dev_span);
/* The output all-gather (a7; H5) fused into the attention epilogues: every
 * later run of this plan stores each final output row not only into `out` but also, at the
 * same element offset (same strides), into outs[0, n) — with kv-head sharding these are the
 * peers' gathered output buffers shifted to this rank's head block, mapped into this process
 * (CUDA IPC / symmetric memory over NVLink), so the gather overlaps the attention tile by tile
 * instead of following it.  Rows that go through partials are stored by the merge kernel.  The
 * caller orders the peers' reads after every rank's run (a cross-rank barrier on the stream).
 * n <= 7 device pointers, 16-byte aligned; n = 0 clears.  lse is written locally only. */
kva_status kva_plan_set_outputs(kva_plan *plan, int32_t n, void *const *outs);
kva_status kva_plan_set_timing_events(kva_plan *plan, void *tile_begin, void *tile_end,
                                      void *decode_begin, void *decode_end);
/* Number of kernel launches hybrid_attention_run_phases(plan, phases) enqueues. */
kva_status kva_plan_launch_count(const kva_plan *plan, int32_t phases, int32_t *n_launches);
/* Plans use the pool's side stream and events: destroy every plan of a pool (and let its
 * enqueued work finish) before kv_pool_destroy. */
kva_status kva_plan_destroy(kva_plan *plan);
/* Plan statistics: counts of work items per kernel and algorithmic bytes/flops. */
typedef struct {
  int64_t n_decode_items, n_tile_items, n_cascade_items, n_merge_rows;  /* decode/merge: per kv head */
  int64_t kv_bytes_algorithmic;     /* distinct KV bytes (prefix once per group/kv-head) */
  int64_t q_bytes, o_bytes;         /* bf16 Q read + O written */
  int64_t decode_kv_bytes;          /* KV bytes read by the split-KV (decode) kernel */
  int64_t flops;                    /* 4*d per (q-head, query, visible key) */
  int64_t tile_flops;               /* the part of `flops` done by the tensor-core tile kernel */
  int64_t host_validate_ns, host_build_ns, host_total_ns;  /* host cost of this plan call */
} kva_plan_stats;
kva_status kva_plan_get_stats(const kva_plan *plan, kva_plan_stats *stats);
kva_status hybrid_attention(kva_pool *pool, const kva_batch_desc *desc, const void *q,
                            int64_t q_stride_tok, int64_t q_stride_head, void *out,
                            int64_t o_stride_tok, int64_t o_stride_head, int32_t out_dtype,
                            float *lse, void *workspace, size_t workspace_bytes,
                            kva_stream_t stream);

/* ------------------------------------------------------------------------------------
 * Eviction (a8).  Block states (S:103 BlockMeta.task_class + reading #17):
 *   0 free, 1 running-online, 2 pinned (referenced by this iteration's batch),
 *   3 active-offline, 4 finished-online, 5 finished-offline.
 * evict_keys: priority_of as an order-preserving u64 key:
 *   free / running-online / pinned -> UINT64_MAX (never selected)
 *   rc > 0 -> priority rc ; finished-online (rc 0) -> 0.5 ; other offline (rc 0) -> 0
 *   code16 = min(2*priority, 0xFFFE);
 *   key = code16 << 48 | lat32 << 16 | (0xFFFF - min(depth, 0xFFFF))      (readings #18-#20)
 *   state, rc, lat, depth: device arrays [n] (uint8, uint32, uint32, uint16; depth nullable
 *   => 0).  Unknown state -> UINT64_MAX and KVA_ERR_INVALID is NOT detected on device.
 * evict_select: the k blocks with the smallest (key, block id), in that order (P:338
 *   "first consider the priority ... then the last access time").
 *   out_ids: device int32 [k].  *n_selected (host) = min(k, #evictable) — this implies one
 *   stream synchronisation; n_selected = NULL enqueues only (no sync, no SHORT status; the
 *   unused tail of out_ids is left untouched), which apply != 0 does not allow.  apply != 0 marks the selected blocks free in free_bits and in
 *   the pool's host mirror (pool required then).  KVA_EVICTION_SHORT if fewer than k.
 *   workspace: evict_select_workspace_size(n, k) bytes of device scratch.
 * ------------------------------------------------------------------------------------ */
/* kv_release_blocks: return blocks to the free pool (recompute-mode preemption or a
 * finished request whose KV is dropped, "preempts and release the KV cache of the
 * victim request").  ids: HOST int32 [n], each allocated (not free) and distinct, else
 * KVA_ERR_INVALID with no change.  Sets the device free bits on `stream` and the mirror. */
kva_status kv_release_blocks(kva_pool *pool, const int32_t *ids, int64_t n, kva_stream_t stream);
/* kv_truncate: shorten requests to their first keep_len[i] tokens (recompute-mode preemption
 * releasing a victim's KV, or the rollback of an iteration's kv_append): the blocks of
 * row i at block indices [cdiv(keep_len[i], 16), cdiv(ctx_len[i], 16)) that are not -1 are
 * returned to the free pool (device free bits + host mirror) and those table entries set to -1
 * in the host mirror AND the device table (one kernel on `stream`, lists as kernel
 * parameters).  keep_len: HOST int32 [num_reqs]; -1 leaves request i untouched, otherwise
 * 0 <= keep_len[i] <= ctx_len[i].  Reads only ctx_len, max_blocks, the tables and the group
 * fields of the descriptor; ctx_len / q_indptr are the caller's to update.  Errors (nothing
 * changed): KVA_ERR_INVALID for a bad keep_len, an id out of range, already free or listed
 * twice; KVA_ERR_GROUP if the cut lies inside the request's shared prefix (its blocks belong
 * to the group). */
kva_status kv_truncate(kva_pool *pool, kva_batch_desc *desc, const int32_t *keep_len, kva_stream_t stream);

enum { KVA_BLK_FREE = 0, KVA_BLK_RUNNING_ONLINE = 1, KVA_BLK_PINNED = 2,
       KVA_BLK_ACTIVE_OFFLINE = 3, KVA_BLK_FINISHED_ONLINE = 4, KVA_BLK_FINISHED_OFFLINE = 5 };

kva_status evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                      const uint16_t *depth, int64_t n, uint64_t *keys_out,
                      kva_stream_t stream);
kva_status evict_select_workspace_size(int64_t n, int64_t k, size_t *bytes);
kva_status evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                        int64_t *n_selected, int32_t apply, kva_pool *pool, void *workspace,
                        size_t workspace_bytes, kva_stream_t stream);

/* ---- KV-manager step (§4.2 "Priority-based KV cache
 * eviction" / "Threshold to limit the KV cache size for active requests") ----
 * One device pass per iteration over the pool's block metadata, feeding evict_select:
 *   1. class transitions (S:161-168 release_request: finished online -> FINISHED_ONLINE,
 *      finished offline -> FINISHED_OFFLINE, preempted offline -> ACTIVE_OFFLINE; reading #17:
 *      this iteration's batch -> RUNNING_ONLINE / PINNED): chain j of the HOST CSR
 *      (chain_indptr, chain_ids) gets state chain_state[j] and lat = now; a block listed in
 *      several chains takes the LAST chain's state (list order);
 *   2. reference counts (S:154-160 update_references; "how may offline requests
 *      (including current running request) will reuse it"), DEVICE id lists (chains
 *      concatenated; order irrelevant):
 *        recount != 0: rc[b] = number of offline-pool chains that list b (pool_ids[0, pool_len));
 *        recount == 0: rc[b] += #chains in pool_ids that list b (requests that joined the
 *                      pool) - #chains in del_ids[0, del_len) that list b (requests that left);
 *                      the caller keeps the counts consistent (a negative count is not
 *                      detected on the device; the oracle reports it as INVALID);
 *   3. *n_active (device int64, nullable) = blocks of the active classes: running
 *      online / pinned, or rc > 0 in any resident class (reading #15);
 *   4. keys_out = evict_keys(state, rc, lat, depth).
 * Host arrays are validated before anything is enqueued (ids in [0, n), states <= 5, indptr
 * monotone from 0 -> else KVA_ERR_INVALID, nothing changed).  Device pool ids outside [0, n)
 * are skipped (not detected).  workspace: kv_manager_step_workspace_size() bytes of device
 * scratch (the deduplicated transition list is uploaded there). */
typedef struct {
  int64_t num_blocks;
  uint8_t *state;          /* device [n] KVA_BLK_* */
  uint32_t *rc;            /* device [n] (rewritten by the recount) */
  uint32_t *lat;           /* device [n] logical ticks (reading #18) */
  const uint16_t *depth;   /* device [n] chain depth (reading #19), nullable */
} kva_block_meta;
typedef struct {
  uint32_t now;
  int32_t n_chains;
  const int32_t *chain_indptr;  /* host [n_chains + 1] */
  const int32_t *chain_ids;     /* host [chain_indptr[n_chains]] */
  const uint8_t *chain_state;   /* host [n_chains] */
  int32_t recount;              /* 1: full recount from pool_ids; 0: incremental */
  const int32_t *pool_ids;      /* device [pool_len] */
  int64_t pool_len;
  const int32_t *del_ids;       /* device [del_len] (incremental mode only) */
  int64_t del_len;
  /* 1: chain_indptr / chain_ids / chain_state are DEVICE arrays (e.g. the finished requests'
   * block-table rows already on the GPU): no upload and no host id check — ids outside
   * [0, num_blocks) are skipped on the device; n_chain_ids (host) = chain_indptr[n_chains]. */
  int32_t chains_on_device;
  int64_t n_chain_ids;
} kva_manager_update;
kva_status kv_manager_step_workspace_size(const kva_block_meta *meta, const kva_manager_update *u,
                                          size_t *bytes);
kva_status kv_manager_step(const kva_block_meta *meta, const kva_manager_update *u,
                           uint64_t *keys_out, int64_t *n_active, void *workspace,
                           size_t workspace_bytes, kva_stream_t stream);
/* kv_manager_step followed by evict_select(keys_out, num_blocks, k, out_ids, n_selected = NULL,
 * apply = 0) — the KV manager's per-iteration pass and its victim order —
 * as ONE cooperative kernel: the manager's key pass writes keys_out and feeds the selection's
 * first pass directly (one launch and one pass over the keys fewer).  Results are identical to
 * the two calls in sequence (keys_out, *n_active, the metadata updates, out_ids[0, min(k, E)));
 * the selected count is left on the device in the first 8 bytes of sel_workspace (int64), as
 * with evict_select's asynchronous mode.  workspace: kv_manager_step_workspace_size();
 * sel_workspace: evict_select_workspace_size(num_blocks, k).  k == 0: the manager step alone.
 * Errors: those of the two calls (validation before anything is enqueued). */
kva_status kv_manager_step_select(const kva_block_meta *meta, const kva_manager_update *u,
                                  uint64_t *keys_out, int64_t *n_active, void *workspace,
                                  size_t workspace_bytes, int64_t k, int32_t *out_ids,
                                  void *sel_workspace, size_t sel_workspace_bytes, kva_stream_t stream);
/* Burst-reserve threshold for kv_append.  threshold_blocks
 * < 0 disables it (default); 0 <= threshold <= num_blocks else KVA_ERR_INVALID.  With a
 * threshold, kv_append first checks capacity (KVA_NEEDS_EVICTION, deficit = need - free),
 * then, if any OFFLINE request (KVA_OFFLINE_PREFILL / KVA_OFFLINE_DECODE) needs a new block:
 * active + need > threshold -> KVA_NEEDS_EVICTION with *deficit = active + need - threshold,
 * nothing changed (online requests may allocate into the reserve; reading R35).  `active` is
 * the last value given to kv_pool_set_active_blocks (e.g. the manager step's n_active) plus
 * the blocks allocated by kv_append since. */
kva_status kv_pool_set_threshold(kva_pool *pool, int64_t threshold_blocks);
kva_status kv_pool_set_active_blocks(kva_pool *pool, int64_t active_blocks);

/* ---- prefix index + batch grouping (host only) ----
 * A block-granular radix index over token ids: one entry per cached block, keyed by (parent
 * entry, the block's 16 token ids), so identical token prefixes map to the same physical
 * blocks ("prefix caching").  Sub-block matches are misses.
 *   kva_prefix_insert: register the whole blocks of tokens[0, n_tokens) with their block ids
 *     (blocks already cached must carry the same id; a new id must not be indexed elsewhere;
 *     else KVA_ERR_INVALID, nothing changed); LAT of the chain = now.
 *   kva_prefix_lookup (S:125-133 lookup_prefix): the longest cached prefix of whole blocks;
 *     *n_hit blocks, the first min(cap, n_hit) ids written to out_block_ids; their LAT = now.
 *   kva_prefix_remove: drop evicted blocks and every entry below them (no dangling
 *     entries S:109); unknown ids are ignored.
 *   kva_group_batch: the batch descriptor's shared-prefix groups from the requests' token ids
 *     (tokens[i][0, n_tokens[i]) = request i's context): usable_i = min(cached prefix blocks,
 *     prefix_limit_blocks[i]) (nullable; pass floor((ctx - q_len)/16) so the queries lie after
 *     the prefix, reading #8).  Requests with usable_i >= min_blocks whose first min_blocks
 *     blocks are the same entries form a group if there are >= 2 of them; its prefix is the
 *     deepest entry all members share, capped by every member's usable_i.  Groups are numbered
 *     in order of their first member; group_of[i] = -1 for the rest.  group_prefix_blocks needs
 *     room for R entries. */
typedef struct kva_prefix_index kva_prefix_index;
kva_status kva_prefix_index_create(kva_prefix_index **out);
kva_status kva_prefix_index_destroy(kva_prefix_index *ix);
kva_status kva_prefix_insert(kva_prefix_index *ix, const int32_t *tokens, int64_t n_tokens,
                             const int32_t *block_ids, uint32_t now);
kva_status kva_prefix_lookup(kva_prefix_index *ix, const int32_t *tokens, int64_t n_tokens,
                             int32_t *out_block_ids, int64_t cap, int64_t *n_hit, uint32_t now);
kva_status kva_prefix_remove(kva_prefix_index *ix, const int32_t *block_ids, int64_t n);
kva_status kva_prefix_size(const kva_prefix_index *ix, int64_t *n_blocks);
kva_status kva_group_batch(kva_prefix_index *ix, int32_t num_reqs, const int32_t *const *tokens,
                           const int64_t *n_tokens, const int32_t *prefix_limit_blocks,
                           int32_t min_blocks, int32_t *group_of, int32_t *group_prefix_blocks,
                           int32_t *num_groups);
/* kva_group_batch_nested: nested groups for the multi-level cascade (group_parent of the batch
 * descriptor).  Level l (thresholds level_min_blocks[] strictly increasing) groups requests whose
 * first level_min_blocks[l] blocks are the same entries; a group's prefix is the deepest entry
 * all its members share (capped by every usable_i); a group whose prefix does not extend its
 * parent's is dropped (its members stay in the parent); group_parent[g] = the nearest kept group
 * above (-1 at the top).  Groups are numbered level by level in order of first member (parents
 * precede children); group_of[i] = request i's deepest group.  Output arrays need R entries. */
kva_status kva_group_batch_nested(kva_prefix_index *ix, int32_t num_reqs, const int32_t *const *tokens,
                                  const int64_t *n_tokens, const int32_t *prefix_limit_blocks,
                                  int32_t n_levels, const int32_t *level_min_blocks,
                                  int32_t *group_of, int32_t *group_prefix_blocks,
                                  int32_t *group_parent, int32_t *num_groups);

/* ---- tuning and diagnostics options (process-wide; read by every later call) ----
 *   "tile_ctas"   persistent CTAs of the tile kernel while it overlaps the decode kernel
 *                 (0 = the planner's split from measured rates, default)
 *   "overlap"     1 = tile kernel concurrent with decode (default), 0 = decode then tile
 *   "pdl"         1 = decode launched as a programmatic dependent of the tile kernel on one
 *                 stream (default), 0 = the two kernels on two streams (events)
 *   "evict_ctas"  CTAs of the cooperative evict_select kernel (0 = #SMs / 2, default)
 *   "evict_threads" 512 (default): the selection's fastest build alone; 256: a build whose CTA
 *                 (~30 KB of shared memory, 256 x 80 registers) shares its SM with two decode
 *                 CTAs — for selections that run beside a long decode-bound attention step
 *                 (same results; other values -> KVA_ERR_INVALID)
 *   "fold"        1: in the one-stream overlapped mode, decode-class members of a one-level
 *                 group whose suffix is one split merge their partial with the group's cascade
 *                 partial in the decode kernel's epilogue (waiting on the tile kernel's
 *                 per-item completion counters) instead of in the merge kernel — bit-identical
 *                 results; 0 (default): the decode kernel then waits for the cascade tiles,
 *                 which measured slower on qwen14b (step period 122 vs 117 us)
 *   "span_ring"   device address of a u64 [5][256][2] ring: manager (0) / evict_select (1) /
 *                 append + allocation (2) / prefill-row append (3) / release (4): launch i
 *                 writes {CTA 0 start, latest CTA end} (%globaltimer ns) at [kind][i % 256]
 *   "host_prof"   1 = accumulate host section times (printed at process exit)
 *   "debug_flags" tile-kernel diagnostics, WRONG RESULTS: 1 = softmax skipped, 2 = PV MMAs not
 *                 issued, 4 = QK MMAs not issued (pipeline studies)
 *   "debug_ts"    device address of a role-timestamp buffer (builds with -DKVA_TILE_TIMESTAMPS)
 * Unknown name -> KVA_ERR_INVALID.  Not synchronised with calls in flight on other threads. */
kva_status kva_set_option(const char *name, int64_t value);
kva_status kva_get_option(const char *name, int64_t *value);
/* ---- diagnostics (not part of the hot path) ----
 * kva_diag_occupy: enqueue n_ctas CTAs that each hold smem_bytes of shared memory and spin
 * for ns nanoseconds on `stream`; a kernel launched right after on another stream then runs on
 * the remaining SMs (profiles/decode_sm_curve.py: decode bandwidth vs SM count). */
kva_status kva_diag_occupy(int32_t n_ctas, int32_t smem_bytes, int64_t ns, kva_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KVATTN_H_ */
