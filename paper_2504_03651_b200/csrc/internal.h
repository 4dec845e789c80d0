// internal.h — host<->device structures and launcher declarations of libkvattn.
// Product code (CUDA path).  Shares nothing with oracle/.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/kvattn.h"

namespace kva {

// sets the thread-local kva_last_error() message (kvattn_host.cu) and returns st
kva_status set_error(kva_status st, const char *msg);

// cudaFuncSetAttribute(max dynamic smem = smem, carveout = max shared) once per (kernel,
// device, smem) — the attribute calls cost microseconds per launch otherwise (kvattn_host.cu)
cudaError_t smem_attrs_once(const void *kern, int smem);
// multiprocessor count of the current device (cached)
int sm_count();

// Tuning / diagnostics options (kva_set_option; process-wide, read at each call)
enum Opt : int { kOptTileCtas = 0, kOptOverlap, kOptPdl, kOptEvictCtas, kOptHostProf, kOptDebugFlags, kOptDebugTs,
                 kOptSpanRing, kOptEvictThreads, kOptFold, kOptCount };
// span_ring (diagnostics): device u64 [5][256][2] — manager (0) / evict_select (1) / append of
// the decode-class rows + allocation (2) / append of the prefill rows (3) / release (4): launch i
// writes [kind][i % 256] = {CTA 0 start, latest CTA end} (%globaltimer ns)
unsigned long long *span_ring_slot(int kind);
#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
int64_t opt(Opt o);

constexpr int kBlock = 16;        // tokens per KV block (reading #5)
constexpr int kSplitKeys = 512;   // fixed split-KV length (depends only on ctx, H9)
constexpr int kDecodeRows = 16;   // rows (q tokens x g heads) one decode warp handles
constexpr int kTileMTc = 128;     // rows per tcgen05 tile CTA (UMMA M = TMEM lanes)
constexpr int kTileN = 64;        // keys per tile-kernel pipeline stage (4 blocks)
constexpr int kMaxOutExtra = 7;   // extra output destinations (peers of an 8-GPU node)

// One decode warp: <= 16 rows (tok*g + hh) of one request and kv-head over keys [k0, k1).
// One decode-class request: keys [kb, ctx) are cut into nsplit splits of
// kSplitKeys; the decode kernel runs every (split, kv head) as one warp.  Partial slot of
// (head h, split s, row r) = slot + (h * nsplit + s) * rows + r, rows = n_tok * g; slot < 0:
// single split, the output is written directly.
// fold: index into the plan's FoldReq list (-1: none) — a decode-class member of a one-level
// group whose suffix is one split: in fold mode the decode kernel merges its own partial with
// the group's cascade partial in its epilogue (no merge-kernel entry)
struct DecodeReq {
  int32_t q_row0, n_tok, table_row, kb, ctx, slot, nsplit, fold;
};
// casc_slot / casc_hstride as in MergeReq (head 0); member_row0: the member's first row in the
// group's stacked row space; flag_base: the group's first cascade-item index (kv head 0), mtiles
// items per kv head (item of row x, head h = flag_base + h * mtiles + x / 256; Q tile (x % 256) / 128)
struct FoldReq {
  int32_t casc_slot, casc_hstride, member_row0, flag_base, mtiles, pad[3];
};

// One tile CTA: <= kTileM rows of one row space (r = tok*g + hh) over keys [k0, k1).
enum : int32_t { kTileList = 1, kTileCausal = 2 };
struct TileItem {
  int32_t row_src;   // contiguous: q row of tok 0; list mode: offset into row_list
  int32_t r0;        // first row index of this tile in the row space
  int32_t n_rows;    // rows in this tile (<= kTileM)
  int32_t kv_head;
  int32_t table_row;
  int32_t k0, k1;
  int32_t pos0;      // causal: position of tok 0
  int32_t slot;      // partial slot of row r0; -1 = direct output
  int32_t flags;     // kTile* bits; bits 8+: cascade item index + 1 (fold completion flags)
};

// One request whose partials are merged (a6): each of its rows r < rows is merged for every
// kv head h (q head = h * g + r % g) from the cascade-prefix slots casc_slot[l] +
// h*casc_hstride[l] + r (l < n_casc, one per nested group level) and the split slots
// split_slot + (h * nsplit + s) * rows + r.
// Nested shared-prefix groups: one cascade partial per level (outermost first).
constexpr int kMaxCascade = 4;
struct MergeReq {
  int32_t q_row0, rows, split_slot, nsplit, n_casc, pad0, pad1, pad2;
  int32_t casc_slot[kMaxCascade], casc_hstride[kMaxCascade];
};

// Request list + exclusive prefix of work units (splits or rows) per request, handed to the
// decode / merge kernels as a __grid_constant__ kernel parameter when n <= kInlineReqs (no
// host->device copy between kv_append and the attention launches), else uploaded with the
// plan (ptr / pre_ptr set).
constexpr int kInlineReqs = 400;
template <class R>
struct ReqList {
  int32_t n;
  const R *ptr;
  const int32_t *pre_ptr;
  int32_t pre[kInlineReqs + 1];
  R req[kInlineReqs];
};

// Per-request append info (kv_append).  blk[0..1]: the ids of blocks pos0/16 and pos0/16 + 1
// when the host resolved them (decode-class requests: <= 16 new tokens, so <= 2 blocks; the
// kernel then reads no table entry and needs no ordering behind the table update), else -1.
struct AppendReq {
  int32_t q_row0, q_len, pos0, table_row, blk[2];
};

struct AttnParams {
  // pool
  const uint16_t *k_pool, *v_pool;
  int32_t num_blocks, Hkv, Hq, g, d;
  const int32_t *block_table;
  int32_t max_blocks;
  float scale_log2;       // sm_scale * log2(e)
  // io
  const uint16_t *q;
  int64_t q_stride_tok, q_stride_head;
  void *out;
  int64_t o_stride_tok, o_stride_head;
  // a7 fused into the epilogues: every output row is also stored at the same element offset in
  // out_extra[0, n_out_extra) — peers' gathered buffers over NVLink (kva_plan_set_outputs)
  int32_t n_out_extra;
  void *out_extra[kMaxOutExtra];
  int32_t out_f32;
  float *lse;             // nullable [total_q][Hq]
  // workspace
  float *part_o;          // [slots][d]
  float *part_lse;        // [slots]
  const int32_t *row_list;
  unsigned long long *dbg;  // optional timestamps (diagnostics; KVA_DEBUG_TS), nullable
  // optional kernel spans (%globaltimer ns): [0] = min decode CTA start, [1] = max decode CTA
  // end, [2] / [3] = the same for the tile kernel, [4] / [5] for the merge kernel
  // (kva_plan_set_span_buffer), nullable
  unsigned long long *span;
  int32_t debug_flags;      // diagnostics only (KVA_DEBUG_FLAGS): 1 = tile softmax skipped
  // fold (decode-epilogue merge of cascade members): FoldReq list, per (cascade item, Q tile)
  // completion counters (+1 per softmax warp, zeroed by the plan upload), this run's epoch
  // (runs that launched the tile kernel, counting this one), fold_on = this run folds
  const FoldReq *fold;
  unsigned *fold_flags;
  uint32_t epoch;
  int32_t fold_on;
};

// launchers (kernels_*.cu)
cudaError_t launch_decode(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                          const ReqList<DecodeReq> &reqs, int n_units, cudaStream_t s, bool pdl = false,
                          const void *tmap_k3 = nullptr, const void *tmap_v3 = nullptr);
// Tile items of the tcgen05 kernel: kernel parameter when n <= kInlineTiles (no upload, so the
// tile kernel is not ordered behind a host->device copy and claims its SMs first), else uploaded.
constexpr int kInlineTiles = 560;
struct TileList {
  int32_t n;
  const TileItem *ptr;
  TileItem item[kInlineTiles];
};
cudaError_t launch_tile_tc2(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                            const TileList &items, int max_ctas, cudaStream_t s,
                            const void *tmap_v3 = nullptr, const void *tmap_k3 = nullptr);
cudaError_t launch_merge(const AttnParams &p, const ReqList<MergeReq> &reqs, int n_units, cudaStream_t s);
// Newly allocated blocks (table entry index, block id): kernel parameter when n <= kInlineAlloc,
// else uploaded (tbl_ptr / ids_ptr set).
constexpr int kInlineAlloc = 1536;
struct AllocList {
  int32_t n;
  const int32_t *tbl_ptr, *ids_ptr;
  int32_t tbl[kInlineAlloc];
  int32_t ids[kInlineAlloc];
};
// Append of a request list; al != nullptr: the same launch also publishes the allocation (table
// entries + free bits) — only for a list whose requests all carry resolved blk ids (it reads
// no table entry), so no ordering between the two parts is needed.
cudaError_t launch_append(const uint16_t *k_new, const uint16_t *v_new, int64_t stride_tok,
                          uint16_t *k_pool, uint16_t *v_pool, int32_t Hkv, int32_t d,
                          int32_t *block_table, int32_t max_blocks,
                          const ReqList<AppendReq> &reqs, int32_t total_new_tok, cudaStream_t s,
                          bool early_trigger = false, const AllocList *al = nullptr,
                          uint32_t *free_bits = nullptr);
cudaError_t launch_evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                              const uint16_t *depth, int64_t n, uint64_t *keys, cudaStream_t s);
cudaError_t launch_manager_step(uint8_t *state, uint32_t *rc, uint32_t *lat, const uint16_t *depth,
                                int64_t n, uint32_t now, const int32_t *tr_ids, int64_t n_tr,
                                const int32_t *tr_indptr, const uint8_t *tr_state, int32_t n_chains,
                                int32_t *win, bool recount, const int32_t *pool_ids, int64_t pool_len,
                                const int32_t *del_ids, int64_t del_len, uint64_t *keys, int64_t *n_active,
                                cudaStream_t s);

// KV-manager step arguments (kernels_evict.cu manager_kernel; kernels_select.cu runs the same
// phases ahead of the selection when fused, kv_manager_step_select)
struct MgrArgs {
  uint8_t *state;
  uint32_t *rc, *lat;
  const uint16_t *depth;
  int64_t n;
  uint32_t now;
  const int32_t *tr_ids;
  int64_t n_tr;
  const int32_t *tr_indptr;
  const uint8_t *tr_state;
  int32_t n_chains;
  int32_t *win;
  int32_t recount;
  const int32_t *pool_ids;
  int64_t pool_len;
  const int32_t *del_ids;
  int64_t del_len;
  uint64_t *keys;
  unsigned long long *n_active;
  unsigned long long *span;  // diagnostics (span_ring): {CTA 0 start, latest CTA end}
};
inline MgrArgs make_mgr_args(uint8_t *state, uint32_t *rc, uint32_t *lat, const uint16_t *depth, int64_t n,
                             uint32_t now, const int32_t *tr_ids, int64_t n_tr, const int32_t *tr_indptr,
                             const uint8_t *tr_state, int32_t n_chains, int32_t *win, bool recount,
                             const int32_t *pool_ids, int64_t pool_len, const int32_t *del_ids, int64_t del_len,
                             uint64_t *keys, int64_t *n_active) {
  return MgrArgs{state, rc, lat, depth, n, now, tr_ids, n_tr, tr_indptr, tr_state, n_chains, win,
                 recount ? 1 : 0, pool_ids, pool_len, del_ids, del_len, keys,
                 reinterpret_cast<unsigned long long *>(n_active), nullptr};
}
#ifdef __CUDACC__
// the eviction key of one block (evict_keys' encoding, readings #18-#20) + the active count
__device__ __forceinline__ uint64_t manager_key(uint32_t s, uint32_t r, uint32_t la, uint32_t dp, unsigned &act) {
  act += (s == 1 || s == 2 || (s >= 3 && s <= 5 && r > 0)) ? 1u : 0u;
  if (s == 0 || s == 1 || s == 2 || s > 5) return ~0ull;
  uint64_t code;
  if (r > 0) code = r >= 0x7FFFu ? 0xFFFEull : 2ull * r;
  else code = (s == 4) ? 1ull : 0ull;
  return (code << 48) | ((uint64_t)la << 16) | (0xFFFFull - (uint64_t)dp);
}
// Manager phases 0-2 over thread t0 of nt (grid-stride), sync() = a grid barrier:
//   phase 0  rc = 0 (recount), win[id] = -1 for listed ids, *n_active = 0
//   phase 1  win[id] = max element index listing id ("last chain wins", reading R36)
//   phase 2  winners apply (state, lat = now); rc += pool chains, -= deleted chains
// Ends with a barrier when phase 2 had work (phase 3, the keys, reads what it wrote).
// s_ind: shared memory for the chain index (the binary search of phase 2: ~10 dependent loads
// per transition, L2 round trips when read from global memory), cap entries; the copy is
// ordered before phase 2 by phase 0's barrier
template <class Sync>
__device__ __forceinline__ void manager_phases(const MgrArgs &a, int64_t t0, int64_t nt, Sync &&sync,
                                               int32_t *s_ind = nullptr, int cap = 0) {
  const int32_t *ind = a.tr_indptr;
  if (s_ind && a.n_tr > 0 && a.n_chains + 1 <= cap) {
    for (int i = threadIdx.x; i <= a.n_chains; i += blockDim.x) s_ind[i] = __ldg(a.tr_indptr + i);
    ind = s_ind;
  }
  if (a.recount) {
    const int64_t n4 = (reinterpret_cast<uintptr_t>(a.rc) & 15) ? 0 : a.n / 4;
    for (int64_t q = t0; q < n4; q += nt) reinterpret_cast<uint4 *>(a.rc)[q] = make_uint4(0, 0, 0, 0);
    for (int64_t b = 4 * n4 + t0; b < a.n; b += nt) a.rc[b] = 0u;
  }
  // transition ids outside [0, n) (possible only for device-resident chains, which the host
  // does not check) are skipped in every phase
  for (int64_t e = t0; e < a.n_tr; e += nt) {
    const int32_t id = a.tr_ids[e];
    if ((uint32_t)id < (uint64_t)a.n) a.win[id] = -1;
  }
  if (a.n_active && t0 == 0) *a.n_active = 0ull;
  sync();  // (also orders the n_active reset before phase 3's adds)
  if (a.n_tr > 0) {
    for (int64_t e = t0; e < a.n_tr; e += nt) {
      const int32_t id = a.tr_ids[e];
      if ((uint32_t)id < (uint64_t)a.n) atomicMax(&a.win[id], (int32_t)e);
    }
    sync();
  }
  const int64_t m = a.n_tr + a.pool_len + a.del_len;
  for (int64_t e = t0; e < m; e += nt) {
    if (e < a.n_tr) {
      const int32_t id = a.tr_ids[e];
      if ((uint32_t)id >= (uint64_t)a.n || a.win[id] != (int32_t)e) continue;  // out of range / a later chain lists it
      int lo = 0, hi = a.n_chains - 1;       // chain j: indptr[j] <= e < indptr[j + 1]
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ind[mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      a.state[id] = a.tr_state[lo];
      a.lat[id] = a.now;
    } else if (e < a.n_tr + a.pool_len) {
      const int32_t id = a.pool_ids[e - a.n_tr];
      if ((uint64_t)id < (uint64_t)a.n) atomicAdd(&a.rc[id], 1u);
    } else {
      const int32_t id = a.del_ids[e - a.n_tr - a.pool_len];
      if ((uint64_t)id < (uint64_t)a.n) atomicSub(&a.rc[id], 1u);
    }
  }
  if (m > 0) sync();
}
#endif
size_t evict_select_ws_bytes(int64_t n, int64_t k);
// evict_select: one cooperative kernel of `ctas` CTAs (<= 0: #SMs / 2); free_bits != nullptr:
// the selected blocks are also marked free (apply)
// mgr != nullptr: the manager step runs first in the same kernel (its keys pass writes
// mgr->keys == keys and feeds the selection's first pass: kv_manager_step_select).  Dispatches
// to the 512- or 256-thread build (option evict_threads); the workspace size covers both.
cudaError_t launch_evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                int64_t *d_count, uint32_t *free_bits, void *ws, size_t ws_bytes,
                                int ctas, cudaStream_t s, const MgrArgs *mgr = nullptr);
size_t evict_select_ws_bytes_512(int64_t n, int64_t k);
size_t evict_select_ws_bytes_256(int64_t n, int64_t k);
cudaError_t launch_evict_select_512(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                    int64_t *d_count, uint32_t *free_bits, void *ws, size_t ws_bytes,
                                    int ctas, cudaStream_t s, const MgrArgs *mgr);
cudaError_t launch_evict_select_256(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                    int64_t *d_count, uint32_t *free_bits, void *ws, size_t ws_bytes,
                                    int ctas, cudaStream_t s, const MgrArgs *mgr);
// an empty kernel launched normally: it completes only after everything before it on the
// stream (ends a run whose last kernel is a programmatic dependent that does not wait)
cudaError_t launch_join(cudaStream_t s);
constexpr int kReleaseBatch = 3800;  // ids (+ table entries) per release launch (kernel parameter)
// free bits of ids_host[0, n) set; tbl_host != nullptr: table[tbl_host[i]] = -1 as well
cudaError_t launch_release_ids(uint32_t *free_bits, const int32_t *ids_host, int n, cudaStream_t s,
                               const int32_t *tbl_host = nullptr, int32_t *table = nullptr);

}  // namespace kva
