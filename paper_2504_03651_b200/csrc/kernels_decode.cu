// kernels_decode.cu — split-KV paged decode attention.
//
// The decode stage "uses the KV cache to generate a single token at a time ... memory-bound
// due to the high frequency of KV cache access"; Eq.(7) P:389-391 models its time
// as gamma*max(L) + delta*mean(L) — the max(L) term is load imbalance that fixed-length
// splits (kSplitKeys, depending only on ctx) remove.
//
// Design (B200): one WARP per work item = (request, kv-head, split of <= 512 keys), rows =
// q_len x g <= 16 packed along the MMA M dimension (GQA heads share the K/V bytes).  Each
// warp streams its split's 16-token blocks (K and V, 2*16*d*2 bytes) through its own
// NST-stage ring in shared memory with 2-D TMA (cp.async.bulk.tensor, 128-B swizzle) and
// one mbarrier per stage; lane 0 is the producer.  QK^T and PV run on mma.sync bf16 with fp32
// accumulation (legacy tensor path: ~10x headroom over what the HBM stream needs, H2);
// softmax is online in fp32 with quad shuffles.  Blocks of the split are looked up once
// (lane j holds block j's id).  Output: normalised partial (O, lse) per split, or the final
// output when the item is the row's only contribution.
#include <cuda.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

// ------------------------------------------------------------------------------------------
// Keys along the MMA M dimension.  For decode the rows (q_len x g <= 16) are few, so
// S^T = K Q^T (M = 16 keys, N = 8 rows, K = d) and O^T = V^T P^T (M = 16 dims, N = 8 rows,
// K = 16 keys) waste at most the N padding instead of 15/16 of M (the rows-along-M layout of
// round 1: twice the MMAs and accumulator registers).  P^T goes from the S^T accumulator layout to the B-operand layout
// with two movmatrix transposes.  The running max is updated lazily (only when it grows by more
// than 2^8 for some row of the warp, FA4-style), so the O rescale is skipped on almost every
// block; masking runs only on blocks that reach the causal diagonal or the split end.  Fewer
// instructions per byte let fewer SMs saturate HBM, which is what the co-scheduled tile
// kernel needs (it runs on the remaining SMs).
template <int D, int NR, int NST, int MINB, bool T3>
__global__ void __launch_bounds__(128, MINB)
    decode_kt_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmk,
                     const __grid_constant__ CUtensorMap tmv, const __grid_constant__ ReqList<DecodeReq> L,
                     int n_units) {
  constexpr int HALVES = D / 64;
  constexpr int KBYTES = 16 * D * 2;  // K (or V) of one block for one head
  constexpr int STAGE = 2 * KBYTES;
  constexpr int KT = D / 16;          // k-steps of S^T = K Q^T
  constexpr int MT = D / 16;          // m-tiles (dims) of O^T
  constexpr int SROW = D + 4;         // padded fp32 row of the output staging tile
  static_assert(NST * STAGE >= NR * 8 * SROW * 4, "staging tile must fit the ring");
  constexpr float kLazy = 8.f;        // rescale only when the max grows by > 2^8
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bars[4][NST];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int unit = blockIdx.x * 4 + warp;  // (item, kv head), head fastest
  __shared__ unsigned int s_done;
  if (p.span) {  // instrumentation: CTA start (%globaltimer ns); the only CTA barrier
    if (threadIdx.x == 0) {
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      atomicMin(&p.span[0], t0);
      s_done = 0u;
    }
    __syncthreads();
  }
  if (unit >= n_units) return;             // no CTA-wide barrier below
  const int item = unit / p.Hkv, kv_head = unit - item * p.Hkv;
  const DecodeReq *reqs = L.ptr ? L.ptr : L.req;
  const int32_t *pre = L.ptr ? L.pre_ptr : L.pre;
  int lo = 0, hi = L.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  const DecodeReq rq = reqs[lo];
  const int split = item - pre[lo];
  const int q_row0 = rq.q_row0, n_tok = rq.n_tok;
  const int k0 = rq.kb + split * kSplitKeys;
  const int k1 = min(rq.ctx, k0 + kSplitKeys);
  const int pos0 = rq.ctx - rq.n_tok;
  const int slot = rq.slot < 0 ? -1 : rq.slot + (kv_head * rq.nsplit + split) * (n_tok * p.g);
  uint8_t *sbase = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  uint8_t *ws = sbase + warp * NST * STAGE;
  uint64_t *bar = bars[warp];
  const int g = p.g;
  const int n_rows = n_tok * g;

  if (lane == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int b0 = k0 / kBlock;
  const int nblk = (k1 + kBlock - 1) / kBlock - b0;  // <= 32
  const int32_t *trow = p.block_table + (int64_t)rq.table_row * p.max_blocks + b0;
  const int my_id = lane < nblk ? __ldg(trow + lane) : 0;
  const int row_base = kv_head * kBlock;

  const uint64_t l2pol = policy_evict_first();
  auto issue = [&](int st, int id) {  // lane 0 only
    uint64_t *b = &bar[st];
    mbar_arrive_expect_tx(b, STAGE);
    const int row = id * p.Hkv * kBlock + row_base;
    uint8_t *dst = ws + st * STAGE;
    // The split-KV stream reads every byte once: it is marked evict-first in L2, so it does not
    // push out what the co-running kernels reuse (the tile kernel's K/V tiles, the eviction
    // selection's keys) — llama7b step 448 -> 433 us (profiles/r01b).  Debug flag 16: normal.
    if constexpr (T3) {  // 3-D maps: one box = the block-head's two halves, same smem layout
      if (!(p.debug_flags & 16)) {
        tma_load_3d_hint(dst, &tmk, b, 0, row, 0, l2pol);
        tma_load_3d_hint(dst + KBYTES, &tmv, b, 0, row, 0, l2pol);
      } else {
        tma_load_3d(dst, &tmk, b, 0, row, 0);
        tma_load_3d(dst + KBYTES, &tmv, b, 0, row, 0);
      }
    } else {
#pragma unroll
      for (int h = 0; h < HALVES; ++h) tma_load_2d_hint(dst + h * 2048, &tmk, b, h * 64, row, l2pol);
#pragma unroll
      for (int h = 0; h < HALVES; ++h) tma_load_2d_hint(dst + KBYTES + h * 2048, &tmv, b, h * 64, row, l2pol);
    }
  };
#pragma unroll
  for (int s = 0; s < NST; ++s) {
    const int id = __shfl_sync(0xffffffffu, my_id, s);
    if (lane == 0 && s < nblk) issue(s, id);
  }

  // Q^T as the B operand: n = row (nt*8 + lane/4), k = dims (lane%4)*2 (+1, +8, +9)
  const int cq = (lane & 3) * 2;
  uint32_t qb[NR][KT][2];
#pragma unroll
  for (int nt = 0; nt < NR; ++nt) {
    const int r = nt * 8 + (lane >> 2);
    const uint32_t *qp = nullptr;
    if (r < n_rows)
      qp = reinterpret_cast<const uint32_t *>(p.q + (int64_t)(q_row0 + r / g) * p.q_stride_tok +
                                              (int64_t)(kv_head * g + r % g) * p.q_stride_head);
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      qb[nt][kk][0] = qp ? __ldg(qp + (kk * 16 + cq) / 2) : 0u;
      qb[nt][kk][1] = qp ? __ldg(qp + (kk * 16 + cq + 8) / 2) : 0u;
    }
  }
  // this thread's rows (accumulator columns): nt*8 + cq + {0, 1}
  float m[NR][2], l[NR][2];
  float o[MT][NR][4];
#pragma unroll
  for (int nt = 0; nt < NR; ++nt) {
    m[nt][0] = m[nt][1] = -CUDART_INF_F;
    l[nt][0] = l[nt][1] = 0.f;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) o[mt][nt][0] = o[mt][nt][1] = o[mt][nt][2] = o[mt][nt][3] = 0.f;
  }
  const float sl2 = p.scale_log2;
  // ldmatrix lane addresses: K as A (row = key, col = dim), V^T as A via .trans
  const int ka_key = (lane & 7) + ((lane >> 3) & 1) * 8, ka_col = (lane >> 4) * 8;
  const int va_key = (lane & 7) + (lane >> 4) * 8, va_col = ((lane >> 3) & 1) * 8;

  int st = 0;
  uint32_t ph = 0;
  for (int j = 0; j < nblk; ++j) {
    const int next_id = __shfl_sync(0xffffffffu, my_id, (j + NST) & 31);
    mbar_wait(&bar[st], ph);
    const uint32_t kb = smem_u32(ws + st * STAGE), vb = kb + KBYTES;
    const int key0 = (b0 + j) * kBlock;
    if (key0 + kBlock > k1) {
      // never-written slots of the last block are NaN-poisoned: zero those V rows
      const int vr = k1 - key0;
      uint8_t *vp = ws + st * STAGE + KBYTES;
      for (int c = lane; c < (16 - vr) * HALVES * 8; c += 32) {
        const int h = c / ((16 - vr) * 8), rem = c % ((16 - vr) * 8);
        const int row = vr + rem / 8, ch = rem % 8;
        *reinterpret_cast<uint4 *>(vp + h * 2048 + row * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
      }
      __syncwarp();
    }
    // S^T = K Q^T: 16 keys x 8*NR rows; even / odd k-steps in independent accumulators
    float s[NR][4], s2[NR][4];
#pragma unroll
    for (int nt = 0; nt < NR; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = s2[nt][e] = 0.f;
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      const int col = kk * 16 + ka_col;
      uint32_t a[4];
      ldsm_x4(kb + (col >> 6) * 2048 + sw128(ka_key, col & 63), a[0], a[1], a[2], a[3]);
#pragma unroll
      for (int nt = 0; nt < NR; ++nt) {
        if (kk & 1) mma_bf16(s2[nt], a, qb[nt][kk][0], qb[nt][kk][1]);
        else mma_bf16(s[nt], a, qb[nt][kk][0], qb[nt][kk][1]);
      }
    }
    // scale (log2 domain) + mask only where a key can be invisible: the split end or the
    // causal diagonal of multi-token rows
    const bool need_mask = key0 + kBlock > k1 || key0 + kBlock - 1 > pos0;
#pragma unroll
    for (int nt = 0; nt < NR; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[nt][e] = (s[nt][e] + s2[nt][e]) * sl2;
    if (need_mask) {
#pragma unroll
      for (int nt = 0; nt < NR; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = key0 + (lane >> 2) + (e >> 1) * 8;
          const int r = nt * 8 + cq + (e & 1);
          const bool ok = key < k1 && key <= pos0 + r / g;
          s[nt][e] = ok ? s[nt][e] : -CUDART_INF_F;
        }
    }
    float mx[NR][2];
    bool grow = false;
#pragma unroll
    for (int nt = 0; nt < NR; ++nt) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float v = fmaxf(s[nt][c], s[nt][c + 2]);
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
        v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
        mx[nt][c] = v;
        grow |= v > m[nt][c] + kLazy;
      }
    }
    if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
      for (int nt = 0; nt < NR; ++nt) {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const float mn = fmaxf(m[nt][c], mx[nt][c]);
          const float a = m[nt][c] == -CUDART_INF_F ? 0.f : fast_exp2(m[nt][c] - mn);
          m[nt][c] = mn;
          l[nt][c] *= a;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            o[mt][nt][c] *= a;
            o[mt][nt][c + 2] *= a;
          }
        }
      }
    }
    uint32_t pb[NR][2];
#pragma unroll
    for (int nt = 0; nt < NR; ++nt) {
      const float bA = m[nt][0] == -CUDART_INF_F ? 0.f : m[nt][0];
      const float bB = m[nt][1] == -CUDART_INF_F ? 0.f : m[nt][1];
      const float p0 = fast_exp2(s[nt][0] - bA), p1 = fast_exp2(s[nt][1] - bB);
      const float p2 = fast_exp2(s[nt][2] - bA), p3 = fast_exp2(s[nt][3] - bB);
      l[nt][0] += p0 + p2;
      l[nt][1] += p1 + p3;
      pb[nt][0] = movmatrix_t(pack_bf16(p0, p1));  // keys 0-7
      pb[nt][1] = movmatrix_t(pack_bf16(p2, p3));  // keys 8-15
    }
    // O^T += V^T P^T
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int col = mt * 16 + va_col;
      uint32_t a[4];
      ldsm_x4_t(vb + (col >> 6) * 2048 + sw128(va_key, col & 63), a[0], a[1], a[2], a[3]);
#pragma unroll
      for (int nt = 0; nt < NR; ++nt) mma_bf16(o[mt][nt], a, pb[nt][0], pb[nt][1]);
    }
    __syncwarp();
    if (lane == 0 && j + NST < nblk) {
      fence_proxy_async();
      issue(st, next_id);
    }
    if (++st == NST) {
      st = 0;
      ph ^= 1u;
    }
  }
  // row sums over the 8 key-lanes
#pragma unroll
  for (int nt = 0; nt < NR; ++nt)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float v = l[nt][c];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      l[nt][c] = v;
    }
  // normalised O through a padded fp32 staging tile (the ring is idle: every issued stage
  // was consumed), then row-contiguous stores
  float *stg = reinterpret_cast<float *>(ws);
  __syncwarp();
#pragma unroll
  for (int nt = 0; nt < NR; ++nt) {
    const float iA = l[nt][0] > 0.f ? 1.f / l[nt][0] : 0.f;
    const float iB = l[nt][1] > 0.f ? 1.f / l[nt][1] : 0.f;
    const int rA = nt * 8 + cq;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int dm = mt * 16 + (lane >> 2);
      stg[rA * SROW + dm] = o[mt][nt][0] * iA;
      stg[(rA + 1) * SROW + dm] = o[mt][nt][1] * iB;
      stg[rA * SROW + dm + 8] = o[mt][nt][2] * iA;
      stg[(rA + 1) * SROW + dm + 8] = o[mt][nt][3] * iB;
    }
  }
  constexpr float kLn2 = 0.6931471805599453f;
  // fold: this member's suffix partial is merged here with its group's cascade partial (the
  // tile kernel, resident before this kernel started, counts each stored Q tile of a cascade
  // item: 4 softmax warps per run) — the merge kernel's arithmetic, in its partial order
  const bool folded = p.fold_on && rq.fold >= 0;
  if (lane < 4) {
#pragma unroll
    for (int nt = 0; nt < NR; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = nt * 8 + cq + c;
        if (r >= n_rows) continue;
        const float lse = l[nt][c] > 0.f ? (m[nt][c] + __log2f(l[nt][c])) * kLn2 : -CUDART_INF_F;
        if (folded) {
          stg[r * SROW + D] = lse;  // the padding column
        } else if (slot < 0) {
          if (p.lse) p.lse[(int64_t)(q_row0 + r / g) * p.Hq + kv_head * g + r % g] = lse;
        } else {
          p.part_lse[slot + r] = lse;
        }
      }
  }
  FoldReq fr{};
  if (folded) {
    fr = p.fold[rq.fold];
    if (lane == 0) {
      const uint32_t target = 4u * p.epoch;
      const int x0 = fr.member_row0, x1 = x0 + n_rows - 1;
      const int f0 = 2 * (fr.flag_base + kv_head * fr.mtiles + x0 / 256) + (x0 % 256) / 128;
      const int f1 = 2 * (fr.flag_base + kv_head * fr.mtiles + x1 / 256) + (x1 % 256) / 128;
      for (int f : {f0, f1}) {
        unsigned spins = 0;
        while (ld_acquire_u32(p.fold_flags + f) < target) {
          __nanosleep(128);
          if (++spins > (1u << 26)) __trap();  // a counter that never arrives: fail, not hang
        }
      }
    }
  }
  __syncwarp();
  constexpr int V = D / 32;  // values per lane per row
  if (folded) {
    for (int r = 0; r < n_rows; ++r) {
      const int cs = fr.casc_slot + kv_head * fr.casc_hstride + r;
      const float lc = __ldcg(p.part_lse + cs), lo = stg[r * SROW + D];
      const float *src = stg + r * SROW + lane * V;
      const float *csrc = p.part_o + (int64_t)cs * D + lane * V;
      const float L = fmaxf(lc, lo);
      const float w0 = lc == -CUDART_INF_F ? 0.f : __expf(lc - L);
      const float w1 = lo == -CUDART_INF_F ? 0.f : __expf(lo - L);
      float sum = 0.f;
      sum += w0;
      sum += w1;
      const float inv = 1.f / sum;
      float v[V];
#pragma unroll
      for (int i = 0; i < V; i += 2) {
        const float2 xc = __ldcg(reinterpret_cast<const float2 *>(csrc + i));
        const float2 xo = *reinterpret_cast<const float2 *>(src + i);
        float a0 = 0.f, a1 = 0.f;
        a0 += w0 * xc.x;
        a1 += w0 * xc.y;
        a0 += w1 * xo.x;
        a1 += w1 * xo.y;
        v[i] = a0 * inv;
        v[i + 1] = a1 * inv;
      }
      const int64_t qrow = q_row0 + r / g;
      const int hq = kv_head * g + r % g;
      const int64_t off = qrow * p.o_stride_tok + hq * p.o_stride_head + lane * V;
      for (int o = 0; o <= p.n_out_extra; ++o) {
        void *base = o == 0 ? p.out : p.out_extra[o - 1];
        if (p.out_f32) {
          float *dst = reinterpret_cast<float *>(base) + off;
#pragma unroll
          for (int i = 0; i < V; i += 2) *reinterpret_cast<float2 *>(dst + i) = make_float2(v[i], v[i + 1]);
        } else {
          uint16_t *dst = reinterpret_cast<uint16_t *>(base) + off;
#pragma unroll
          for (int i = 0; i < V; i += 2) *reinterpret_cast<uint32_t *>(dst + i) = pack_bf16(v[i], v[i + 1]);
        }
      }
      if (p.lse && lane == 0) p.lse[qrow * p.Hq + hq] = L + __logf(sum);
    }
  }
  for (int r = 0; r < (folded ? 0 : n_rows); ++r) {
    const float *src = stg + r * SROW + lane * V;
    float v[V];
#pragma unroll
    for (int i = 0; i < V; i += 2) {
      const float2 t = *reinterpret_cast<const float2 *>(src + i);
      v[i] = t.x;
      v[i + 1] = t.y;
    }
    if (slot < 0) {
      const int64_t qrow = q_row0 + r / g;
      const int hq = kv_head * g + r % g;
      const int64_t off = qrow * p.o_stride_tok + hq * p.o_stride_head + lane * V;
      for (int o = 0; o <= p.n_out_extra; ++o) {  // own output, then the peers' (fused a7)
        void *base = o == 0 ? p.out : p.out_extra[o - 1];
        if (p.out_f32) {
          float *dst = reinterpret_cast<float *>(base) + off;
#pragma unroll
          for (int i = 0; i < V; i += 2) *reinterpret_cast<float2 *>(dst + i) = make_float2(v[i], v[i + 1]);
        } else {
          uint16_t *dst = reinterpret_cast<uint16_t *>(base) + off;
#pragma unroll
          for (int i = 0; i < V; i += 2) *reinterpret_cast<uint32_t *>(dst + i) = pack_bf16(v[i], v[i + 1]);
        }
      }
    } else {
      float *dst = p.part_o + (int64_t)(slot + r) * D + lane * V;
#pragma unroll
      for (int i = 0; i < V; i += 2) *reinterpret_cast<float2 *>(dst + i) = make_float2(v[i], v[i + 1]);
    }
  }
  if (p.span) {  // instrumentation: the CTA's last active warp records the end
    __syncwarp();
    const int active = min(4, n_units - (int)blockIdx.x * 4);
    if (lane == 0) {
      unsigned long long t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (atomicAdd(&s_done, 1u) == (unsigned)(active - 1)) atomicMax(&p.span[1], t1);
    }
  }
}

template <int D, int NR, int NST, int MINB, bool T3 = false>
static cudaError_t launch_decode_kt(const AttnParams &p, const void *tmk, const void *tmv,
                                   const ReqList<DecodeReq> &L, int n, cudaStream_t s, bool pdl) {
  const size_t smem = 4 * NST * (2 * 16 * D * 2) + 1024;
  auto kern = decode_kt_kernel<D, NR, NST, MINB, T3>;
  // max dynamic smem + full carveout (CTAs of concurrently running kernels share SMs), once
  cudaError_t e = smem_attrs_once(reinterpret_cast<const void *>(kern), (int)smem);
  if (e != cudaSuccess) return e;
  const CUtensorMap &mk = *reinterpret_cast<const CUtensorMap *>(tmk);
  const CUtensorMap &mv = *reinterpret_cast<const CUtensorMap *>(tmv);
  if (!pdl) {
    kern<<<(n + 3) / 4, 128, smem, s>>>(p, mk, mv, L, n);
    return cudaGetLastError();
  }
  // dependent launch: may start while the preceding tile kernel runs (after all its CTAs are
  // resident, griddepcontrol.launch_dependents); no data dependency between the two
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + 3) / 4);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p, mk, mv, L, n);
}

cudaError_t launch_decode(const AttnParams &p, const void *tmk, const void *tmv,
                          const ReqList<DecodeReq> &L, int n, cudaStream_t s, bool pdl,
                          const void *tmk3, const void *tmv3) {
  if (n <= 0) return cudaSuccess;
  int max_rows = 0;
  const DecodeReq *reqs = L.ptr ? nullptr : L.req;
  if (reqs)
    for (int i = 0; i < L.n; ++i) max_rows = std::max(max_rows, reqs[i].n_tok * p.g);
  else
    max_rows = kDecodeRows;
  const bool nr1 = max_rows <= 8;  // one 8-row MMA N tile
  if (p.d == 128 && tmk3 && tmv3)  // one 3-D TMA box per block-head
    return nr1 ? launch_decode_kt<128, 1, 3, 4, true>(p, tmk3, tmv3, L, n, s, pdl)
               : launch_decode_kt<128, 2, 3, 2, true>(p, tmk3, tmv3, L, n, s, pdl);
  if (p.d == 128) return cudaErrorInvalidValue;  // the pool always has the 3-D maps for d = 128
  return nr1 ? launch_decode_kt<64, 1, 4, 2>(p, tmk, tmv, L, n, s, pdl)
             : launch_decode_kt<64, 2, 4, 2>(p, tmk, tmv, L, n, s, pdl);
}

}  // namespace kva
