// internal.h — host<->device structures and launcher declarations of libkvattn.
// Product code (CUDA path).  Shares nothing with oracle/.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace kva {

constexpr int kBlock = 16;        // tokens per KV block (reading #5)
constexpr int kSplitKeys = 512;   // fixed split-KV length (depends only on ctx, H9)
constexpr int kDecodeRows = 16;   // rows (q tokens x g heads) one decode warp handles
constexpr int kTileMMma = 64;     // rows per legacy mma.sync tile CTA (4 warps x 16)
constexpr int kTileMTc = 128;     // rows per tcgen05 tile CTA (UMMA M = TMEM lanes)
constexpr int kTileN = 64;        // keys per tile-kernel pipeline stage (4 blocks)

// One decode warp: <= 16 rows (tok*g + hh) of one request and kv-head over keys [k0, k1).
struct DecodeItem {
  int32_t q_row0;    // first q row of the request
  int32_t n_tok;     // q_len (rows = n_tok * g <= 16)
  int32_t kv_head;   // local kv head
  int32_t table_row; // row of the device block table
  int32_t k0, k1;    // key range (k0 multiple of 16)
  int32_t pos0;      // absolute position of token 0 (ctx - q_len)
  int32_t slot;      // partial slot of row 0 (rows consecutive); -1 = write output directly
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
  int32_t flags;
};

struct MergeRow {
  int32_t q_row, q_head, s_begin, s_count;
};

// Per-request append info (kv_append).
struct AppendReq {
  int32_t q_row0, q_len, pos0, table_row;
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
  int32_t out_f32;
  float *lse;             // nullable [total_q][Hq]
  // workspace
  float *part_o;          // [slots][d]
  float *part_lse;        // [slots]
  const int32_t *row_list;
  unsigned long long *dbg;  // optional timestamps (diagnostics; KVA_DEBUG_TS), nullable
  int32_t debug_flags;      // diagnostics only (KVA_DEBUG_FLAGS): 1 = tile softmax skipped
};

// launchers (kernels_*.cu)
cudaError_t launch_decode(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                          const DecodeItem *items, int n_items, cudaStream_t s);
cudaError_t launch_tile(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                        const TileItem *items, int n_items, cudaStream_t s);
cudaError_t launch_tile_tc(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                           const TileItem *items, int n_items, int max_ctas, cudaStream_t s);
cudaError_t launch_tile_tc2(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                            const TileItem *items, int n_items, int max_ctas, cudaStream_t s);
cudaError_t launch_tile_tc3(const AttnParams &p, const void *tmap_k, const void *tmap_v,
                            const TileItem *items, int n_items, int max_ctas, cudaStream_t s);
cudaError_t launch_merge(const AttnParams &p, const MergeRow *rows, const int32_t *slots,
                         int n_rows, cudaStream_t s);
cudaError_t launch_alloc_write(int32_t *block_table, uint32_t *free_bits, const int32_t *tbl_idx,
                               const int32_t *ids, int32_t n, cudaStream_t s);
cudaError_t launch_append(const uint16_t *k_new, const uint16_t *v_new, int64_t stride_tok,
                          uint16_t *k_pool, uint16_t *v_pool, int32_t Hkv, int32_t d,
                          const int32_t *block_table, int32_t max_blocks, const AppendReq *reqs,
                          const int32_t *q_indptr, int32_t num_reqs, int32_t total_new_tok,
                          cudaStream_t s);
cudaError_t launch_evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                              const uint16_t *depth, int64_t n, uint64_t *keys, cudaStream_t s);
size_t evict_select_ws_bytes(int64_t n, int64_t k);
cudaError_t launch_evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                int64_t *d_count, void *ws, size_t ws_bytes, cudaStream_t s);
constexpr int kReleaseBatch = 4000;  // ids per release launch (kernel-parameter payload)
cudaError_t launch_release_ids(uint32_t *free_bits, const int32_t *ids_host, int n, cudaStream_t s);
cudaError_t launch_free_ids(uint32_t *free_bits, const int32_t *ids, const int64_t *d_count,
                            int64_t k, cudaStream_t s);

}  // namespace kva
