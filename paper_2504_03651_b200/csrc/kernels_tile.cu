// kernels_tile.cu — tiled attention for prefill chunks and shared-prefix (cascade) tiles
// (SURVEY §8(a) a3 + a5), legacy-tensor-core version (mma.sync bf16, fp32 accumulate).
//
// Prefill is "compute-bound" with attention cost "quadratic to the sequence length"
// (Eq.(6)); chunked prefills are batched with decodes.  A CTA owns
// one M-tile of kTileM rows (r = tok*g + hh: GQA heads of a token share K/V) and streams the
// keys [k0, k1) in stages of kTileN keys (4 blocks) through an NST-deep TMA ring (2-D TMA,
// 128-B swizzle, mbarrier complete_tx).  Rows come either from one request (contiguous q
// rows, causal mask by absolute position) or, for a shared-prefix group, from a row list of
// all decode-class members ("cascade": the group's prefix blocks are read once per
// (group, kv-head, M-tile) instead of once per member).
// Output: final O/lse (direct) or a normalised partial merged later by log-sum-exp.
// The tcgen05/TMEM version of this kernel lives in kernels_tile_tc.cu.
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

template <int D, int NST>
__global__ void __launch_bounds__(128, 2)
    tile_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmk,
                const __grid_constant__ CUtensorMap tmv, const TileItem *__restrict__ items) {
  constexpr int HALVES = D / 64;
  constexpr int KBYTES = 16 * D * 2;            // one block, one head
  constexpr int NBLK = kTileN / kBlock;         // 4 blocks per stage
  constexpr int STAGE = 2 * NBLK * KBYTES;      // K then V
  constexpr int KT = D / 16, NT = D / 8, ST = kTileN / 8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t bars[NST];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  const TileItem it = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.g;
  const bool is_list = it.flags & kTileList, causal = it.flags & kTileCausal;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const int b0 = it.k0 / kBlock;
  const int nkb = (it.k1 + kBlock - 1) / kBlock - b0;  // key blocks
  const int nst = (nkb + NBLK - 1) / NBLK;             // stages
  const int32_t *trow = p.block_table + (int64_t)it.table_row * p.max_blocks + b0;

  auto issue = [&](int st, int t) {  // warp 0, all lanes call; lane 0 issues
    const int jb = t * NBLK + (lane & (NBLK - 1));
    const int id = (lane < NBLK && jb < nkb) ? __ldg(trow + jb) : 0;
    const int nb = min(NBLK, nkb - t * NBLK);
    int ids[NBLK];
#pragma unroll
    for (int q = 0; q < NBLK; ++q) ids[q] = __shfl_sync(0xffffffffu, id, q);
    if (lane == 0) {
      uint64_t *b = &bars[st];
      mbar_arrive_expect_tx(b, nb * 2 * KBYTES);
      uint8_t *dst = smem + st * STAGE;
#pragma unroll
      for (int q = 0; q < NBLK; ++q) {
        if (q < nb) {
          const int row = (ids[q] * p.Hkv + it.kv_head) * kBlock;
#pragma unroll
          for (int h = 0; h < HALVES; ++h) {
            tma_load_2d(dst + q * KBYTES + h * 2048, &tmk, b, h * 64, row);
            tma_load_2d(dst + NBLK * KBYTES + q * KBYTES + h * 2048, &tmv, b, h * 64, row);
          }
        }
      }
    }
  };
  if (warp == 0) {
    for (int s = 0; s < NST && s < nst; ++s) issue(s, s);
  }

  // ---- Q fragments for this warp's 16 rows ----
  const int r_lo = it.r0 + warp * 16 + (lane >> 2), r_hi = r_lo + 8;
  const int r_end = it.r0 + it.n_rows;
  const int cq = (lane & 3) * 2;
  auto qrow_of = [&](int r) -> int {
    const int tok = r / g;
    return is_list ? __ldg(p.row_list + it.row_src + tok) : it.row_src + tok;
  };
  uint32_t qa[KT][4];
  int qrow_lo = -1, qrow_hi = -1;
  {
    const uint32_t *qlo = nullptr, *qhi = nullptr;
    if (r_lo < r_end) {
      qrow_lo = qrow_of(r_lo);
      qlo = reinterpret_cast<const uint32_t *>(p.q + (int64_t)qrow_lo * p.q_stride_tok +
                                               (int64_t)(it.kv_head * g + r_lo % g) * p.q_stride_head);
    }
    if (r_hi < r_end) {
      qrow_hi = qrow_of(r_hi);
      qhi = reinterpret_cast<const uint32_t *>(p.q + (int64_t)qrow_hi * p.q_stride_tok +
                                               (int64_t)(it.kv_head * g + r_hi % g) * p.q_stride_head);
    }
#pragma unroll
    for (int kk = 0; kk < KT; ++kk) {
      const int c = kk * 16 + cq;
      qa[kk][0] = qlo ? __ldg(qlo + c / 2) : 0u;
      qa[kk][1] = qhi ? __ldg(qhi + c / 2) : 0u;
      qa[kk][2] = qlo ? __ldg(qlo + (c + 8) / 2) : 0u;
      qa[kk][3] = qhi ? __ldg(qhi + (c + 8) / 2) : 0u;
    }
  }
  const int pos_lo = causal ? it.pos0 + r_lo / g : INT32_MAX;
  const int pos_hi = causal ? it.pos0 + r_hi / g : INT32_MAX;

  float o[NT][4];
#pragma unroll
  for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_lo = -CUDART_INF_F, m_hi = -CUDART_INF_F, l_lo = 0.f, l_hi = 0.f;
  const float sl2 = p.scale_log2;

  for (int t = 0; t < nst; ++t) {
    const int st = t % NST;
    mbar_wait(&bars[st], (t / NST) & 1);
    const int key0 = (b0 + t * NBLK) * kBlock;
    uint8_t *stage = smem + st * STAGE;
    if (key0 + kTileN > it.k1) {
      // zero V rows of keys >= k1 (NaN poison / unloaded blocks) before PV
      const int vr = it.k1 - key0;  // valid keys in this stage, 1..63
      const int nchunk = (kTileN - vr) * HALVES * 8;
      for (int c = threadIdx.x; c < nchunk; c += blockDim.x) {
        const int key = vr + c / (HALVES * 8);
        const int rem = c % (HALVES * 8);
        const int h = rem / 8, ch = rem % 8;
        *reinterpret_cast<uint4 *>(stage + NBLK * KBYTES + (key / 16) * KBYTES + h * 2048 +
                                   (key % 16) * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
      }
      __syncthreads();
    }
    const uint32_t kb = smem_u32(stage), vb = kb + NBLK * KBYTES;
    float s[ST][4];
#pragma unroll
    for (int n = 0; n < ST; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
    {
      const int keyl = (lane >> 4) * 8 + (lane & 7);
      const int csub = ((lane >> 3) & 1) * 8;
#pragma unroll
      for (int kk = 0; kk < KT; ++kk) {
        const int col = kk * 16 + csub;
#pragma unroll
        for (int n2 = 0; n2 < ST / 2; ++n2) {  // 16 keys = one block
          uint32_t r0, r1, r2, r3;
          ldsm_x4(kb + n2 * KBYTES + (col >> 6) * 2048 + sw128(keyl, col & 63), r0, r1, r2, r3);
          mma_bf16(s[2 * n2], qa[kk], r0, r1);
          mma_bf16(s[2 * n2 + 1], qa[kk], r2, r3);
        }
      }
    }
    float mx_lo = -CUDART_INF_F, mx_hi = -CUDART_INF_F;
    const bool need_mask = (key0 + kTileN > it.k1) || (causal && key0 + kTileN - 1 > min(pos_lo, pos_hi));
#pragma unroll
    for (int n = 0; n < ST; ++n) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (need_mask) {
          const int key = key0 + n * 8 + cq + (e & 1);
          const int pos = (e >> 1) ? pos_hi : pos_lo;
          const bool ok = key < it.k1 && key <= pos;
          s[n][e] = ok ? s[n][e] * sl2 : -CUDART_INF_F;
        } else {
          s[n][e] *= sl2;
        }
      }
      mx_lo = fmaxf(mx_lo, fmaxf(s[n][0], s[n][1]));
      mx_hi = fmaxf(mx_hi, fmaxf(s[n][2], s[n][3]));
    }
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 1));
    mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, 2));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 1));
    mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, 2));
    const float mn_lo = fmaxf(m_lo, mx_lo), mn_hi = fmaxf(m_hi, mx_hi);
    const float base_lo = mn_lo == -CUDART_INF_F ? 0.f : mn_lo;
    const float base_hi = mn_hi == -CUDART_INF_F ? 0.f : mn_hi;
    const float a_lo = fast_exp2(m_lo - base_lo), a_hi = fast_exp2(m_hi - base_hi);
    m_lo = mn_lo;
    m_hi = mn_hi;
    float ps_lo = 0.f, ps_hi = 0.f;
#pragma unroll
    for (int n = 0; n < ST; ++n) {
      s[n][0] = fast_exp2(s[n][0] - base_lo);
      s[n][1] = fast_exp2(s[n][1] - base_lo);
      s[n][2] = fast_exp2(s[n][2] - base_hi);
      s[n][3] = fast_exp2(s[n][3] - base_hi);
      ps_lo += s[n][0] + s[n][1];
      ps_hi += s[n][2] + s[n][3];
    }
    l_lo = l_lo * a_lo + ps_lo;
    l_hi = l_hi * a_hi + ps_hi;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      o[n][0] *= a_lo;
      o[n][1] *= a_lo;
      o[n][2] *= a_hi;
      o[n][3] *= a_hi;
    }
    {
      const int keyl = (lane & 7) + ((lane >> 3) & 1) * 8;
      const int csub = (lane >> 4) * 8;
#pragma unroll
      for (int kc = 0; kc < kTileN / 16; ++kc) {  // 16-key chunk = block kc
        uint32_t pa[4];
        pa[0] = pack_bf16(s[2 * kc][0], s[2 * kc][1]);
        pa[1] = pack_bf16(s[2 * kc][2], s[2 * kc][3]);
        pa[2] = pack_bf16(s[2 * kc + 1][0], s[2 * kc + 1][1]);
        pa[3] = pack_bf16(s[2 * kc + 1][2], s[2 * kc + 1][3]);
#pragma unroll
        for (int c16 = 0; c16 < D / 16; ++c16) {
          const int col = c16 * 16 + csub;
          uint32_t r0, r1, r2, r3;
          ldsm_x4_t(vb + kc * KBYTES + (col >> 6) * 2048 + sw128(keyl, col & 63), r0, r1, r2, r3);
          mma_bf16(o[2 * c16], pa, r0, r1);
          mma_bf16(o[2 * c16 + 1], pa, r2, r3);
        }
      }
    }
    __syncthreads();  // stage consumed by all warps
    if (warp == 0 && t + NST < nst) {
      if (lane == 0) fence_proxy_async();
      issue(st, t + NST);
    }
  }
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 1);
  l_lo += __shfl_xor_sync(0xffffffffu, l_lo, 2);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 1);
  l_hi += __shfl_xor_sync(0xffffffffu, l_hi, 2);

  constexpr float kLn2 = 0.6931471805599453f;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int r = half ? r_hi : r_lo;
    if (r >= r_end) continue;
    const float l = half ? l_hi : l_lo, m = half ? m_hi : m_lo;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const float lse = l > 0.f ? (m + __log2f(l)) * kLn2 : -CUDART_INF_F;
    const int hq = it.kv_head * g + r % g;
    if (it.slot < 0) {
      const int64_t qrow = half ? qrow_hi : qrow_lo;
      if (p.out_f32) {
        float *dst = reinterpret_cast<float *>(p.out) + qrow * p.o_stride_tok + hq * p.o_stride_head;
#pragma unroll
        for (int n = 0; n < NT; ++n)
          *reinterpret_cast<float2 *>(dst + n * 8 + cq) =
              make_float2(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
      } else {
        uint16_t *dst =
            reinterpret_cast<uint16_t *>(p.out) + qrow * p.o_stride_tok + hq * p.o_stride_head;
#pragma unroll
        for (int n = 0; n < NT; ++n)
          *reinterpret_cast<uint32_t *>(dst + n * 8 + cq) =
              pack_bf16(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
      }
      if (p.lse && (lane & 3) == 0) p.lse[qrow * p.Hq + hq] = lse;
    } else {
      float *dst = p.part_o + (int64_t)(it.slot + (r - it.r0)) * D;
#pragma unroll
      for (int n = 0; n < NT; ++n)
        *reinterpret_cast<float2 *>(dst + n * 8 + cq) =
            make_float2(o[n][2 * half] * inv, o[n][2 * half + 1] * inv);
      if ((lane & 3) == 0) p.part_lse[it.slot + (r - it.r0)] = lse;
    }
  }
}

template <int D, int NST>
static cudaError_t launch_tile_t(const AttnParams &p, const void *tmk, const void *tmv,
                                 const TileItem *items, int n, cudaStream_t s) {
  const size_t smem = NST * (2 * (kTileN / kBlock) * 16 * D * 2) + 1024;
  auto kern = tile_kernel<D, NST>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // full shared-memory carveout so CTAs of concurrently running kernels can share an SM
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  kern<<<n, 128, smem, s>>>(p, *reinterpret_cast<const CUtensorMap *>(tmk),
                            *reinterpret_cast<const CUtensorMap *>(tmv), items);
  return cudaGetLastError();
}

cudaError_t launch_tile(const AttnParams &p, const void *tmk, const void *tmv,
                        const TileItem *items, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (p.d == 128) return launch_tile_t<128, 3>(p, tmk, tmv, items, n, s);
  return launch_tile_t<64, 4>(p, tmk, tmv, items, n, s);
}

}  // namespace kva
