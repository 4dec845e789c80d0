// kernels_tile_tc.cu — tcgen05/TMEM tiled attention for prefill chunks and shared-prefix
// (cascade) tiles (SURVEY §8(a) a3 + a5): the dense contractions of the mixed batch.
//
// Prefill is "compute-bound", its attention cost "quadratic to the sequence length"
// (Eq.(6)); chunked prefills are batched with memory-bound decodes.
//
// One CTA = one M-tile of 128 query rows (r = tok*g + hh; GQA heads of a token share K/V),
// streaming keys [k0, k1) in N=128-key tiles (8 paged blocks).  Warp roles (192 threads):
//   warp 0      TMA producer: K and V tiles of 8 blocks each (2-D TMA, 128-B swizzle) into a
//               2-stage ring; full/empty mbarriers.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//               S_j = Q K_j^T  (M=128, N=128, K=d; A,B K-major)  -> TMEM S[j&1]
//               O  += P_j V_j  (M=128, N=d, K=128; A K-major, B = V MN-major) -> TMEM O
//   warps 2..5  softmax: one thread per row (= TMEM lane) reads S with tcgen05.ld, masks
//               (causal / key range), online softmax in the log2 domain with lazy O
//               rescaling (only when the row max grows by > 8, i.e. 2^8), writes P (bf16)
//               into shared memory in the UMMA K-major SW128 layout; epilogue O/l from TMEM.
// TMEM columns: S0 [0,128), S1 [128,256), O [256, 256+d).
#include <cuda.h>
#include <math_constants.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

namespace tc {

constexpr int M = 128;          // rows per tile (UMMA M, TMEM lanes)
constexpr int N = 128;          // keys per tile (UMMA N of QK^T, K of PV)
constexpr int NBLK = N / kBlock;  // 8 paged blocks per key tile

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
// kind::f16 instruction descriptor: D f32, A/B bf16, A K-major, B K- or MN-major.
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id,
                                     uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 columns of 32-bit: thread i of the warp gets lane (base+i), 32 columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
}

// byte offset of element (row, col) in a K-major SW128 tile stored as [col/64][rows][64]
__device__ __forceinline__ uint32_t kmaj_off(int row, int col, int rows) {
  return (col >> 6) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
         ((((col & 63) >> 3) ^ (row & 7)) << 4) + ((col & 7) << 1);
}

}  // namespace tc

template <int D>
__global__ void __launch_bounds__(192, 1)
    tile_tc_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmk,
                   const __grid_constant__ CUtensorMap tmv, const TileItem *__restrict__ items,
                   int n_items) {
  using namespace tc;
  constexpr int HALVES = D / 64;
  constexpr int KBYTES = 16 * D * 2;        // one paged block, one head (K or V)
  constexpr int TBYTES = N * D * 2;         // a K or V tile (128 keys)
  constexpr int QBYTES = M * D * 2;
  constexpr uint32_t ID_QK = idesc(M, N, false);
  constexpr uint32_t ID_PV = idesc(M, D, true);
  constexpr uint32_t TM_O = 256;            // TMEM column of O

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;
  uint8_t *sK = sQ + QBYTES;                // [2][TBYTES]
  uint8_t *sV = sK + 2 * TBYTES;            // [2][TBYTES]
  uint8_t *sP = sV + 2 * TBYTES;            // [M*N*2]
  __shared__ uint64_t bar_q, bar_fk[2], bar_fv[2], bar_empty[2], bar_sfull[2], bar_sfree[2], bar_p, bar_o;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.g;
  auto ntiles = [&](const TileItem &t) {
    return ((t.k1 + kBlock - 1) / kBlock - t.k0 / kBlock + NBLK - 1) / NBLK;
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar_q, 128);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bar_fk[s], 1);
      mbar_init(&bar_fv[s], 1);
      mbar_init(&bar_empty[s], 1);
      mbar_init(&bar_sfull[s], 1);
      mbar_init(&bar_sfree[s], 128);
    }
    mbar_init(&bar_p, 128);
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;

  // Persistent: this CTA processes items blockIdx.x, +gridDim.x, ... (LPT-sorted by the
  // planner).  J counts key tiles across items; every barrier phase derives from J (or the
  // item ordinal I for bar_q), identically in every role.
  if (warp == 0) {
    // ------------------------------- TMA producer -------------------------------
    int J = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const TileItem it = items[item];
      const int kb0 = it.k0 / kBlock;
      const int nkb = (it.k1 + kBlock - 1) / kBlock - kb0;
      const int nt = ntiles(it);
      const int32_t *trow = p.block_table + (int64_t)it.table_row * p.max_blocks + kb0;
      for (int j = 0; j < nt; ++j, ++J) {
        const int s = J & 1;
        const int jb = j * NBLK + (lane & (NBLK - 1));
        const int id = (lane < NBLK && jb < nkb) ? __ldg(trow + jb) : 0;
        const int nb = min(NBLK, nkb - j * NBLK);
        int ids[NBLK];
#pragma unroll
        for (int q = 0; q < NBLK; ++q) ids[q] = __shfl_sync(0xffffffffu, id, q);
        if (J >= 2) mbar_wait(&bar_empty[s], ((J >> 1) - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bar_fk[s], nb * KBYTES);
#pragma unroll
          for (int q = 0; q < NBLK; ++q)
            if (q < nb) {
              const int row = (ids[q] * p.Hkv + it.kv_head) * kBlock;
#pragma unroll
              for (int h = 0; h < HALVES; ++h)
                tma_load_2d(sK + s * TBYTES + h * (N * 128) + q * 2048, &tmk, &bar_fk[s], h * 64, row);
            }
          mbar_arrive_expect_tx(&bar_fv[s], nb * KBYTES);
#pragma unroll
          for (int q = 0; q < NBLK; ++q)
            if (q < nb) {
              const int row = (ids[q] * p.Hkv + it.kv_head) * kBlock;
#pragma unroll
              for (int h = 0; h < HALVES; ++h)
                tma_load_2d(sV + s * TBYTES + h * (N * 128) + q * 2048, &tmv, &bar_fv[s], h * 64, row);
            }
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer -------------------------------
    if (lane == 0) {
      const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV),
                     p_base = smem_u32(sP);
      auto issue_pv = [&](int Jg, bool first) {
        const int s = Jg & 1;
        mbar_wait(&bar_p, Jg & 1);
        mbar_wait(&bar_fv[s], (Jg >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < N / 16; ++k) {
          const uint64_t a = sdesc(p_base + (k >> 2) * (M * 128) + (k & 3) * 32, 16, 1024);
          const uint64_t b = sdesc(v_base + s * TBYTES + k * 2048, N * 128, 1024);
          umma(tmem + TM_O, a, b, ID_PV, (!first || k > 0) ? 1u : 0u);
        }
        umma_commit(&bar_o);
        umma_commit(&bar_empty[s]);
      };
      int J = 0, I = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++I) {
        const int nt = ntiles(items[item]);
        mbar_wait(&bar_q, I & 1);
        tc_fence_after();
        for (int j = 0; j < nt; ++j, ++J) {
          const int s = J & 1, b = J & 1;
          mbar_wait(&bar_fk[s], (J >> 1) & 1);
          if (J >= 2) mbar_wait(&bar_sfree[b], ((J >> 1) - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t a = sdesc(q_base + (k >> 2) * (M * 128) + (k & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(k_base + s * TBYTES + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
            umma(tmem + b * N, a, bd, ID_QK, k > 0 ? 1u : 0u);
          }
          umma_commit(&bar_sfull[b]);
          if (j >= 1) issue_pv(J - 1, j == 1);
        }
        issue_pv(J - 1, nt == 1);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------- softmax warps -------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;   // TMEM lane = tile row
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    int J = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const TileItem it = items[item];
      const bool is_list = it.flags & kTileList, causal = it.flags & kTileCausal;
      const int nt = ntiles(it);
      const int r = it.r0 + row;
      const bool valid = r < it.r0 + it.n_rows;
      // Q row -> shared memory (K-major SW128).  Safe: the previous item's last PV (and so
      // every MMA reading Q) completed before this thread's previous epilogue returned.
      int qrow = 0;
      if (valid) {
        const int tok = r / g;
        qrow = is_list ? __ldg(p.row_list + it.row_src + tok) : it.row_src + tok;
        const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (int64_t)qrow * p.q_stride_tok +
                                                           (int64_t)(it.kv_head * g + r % g) * p.q_stride_head);
#pragma unroll
        for (int c = 0; c < D / 8; ++c)
          *reinterpret_cast<uint4 *>(sQ + kmaj_off(row, c * 8, M)) = __ldg(src + c);
      } else {
#pragma unroll
        for (int c = 0; c < D / 8; ++c)
          *reinterpret_cast<uint4 *>(sQ + kmaj_off(row, c * 8, M)) = make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();
      mbar_arrive(&bar_q);

      const int pos = (causal && valid) ? it.pos0 + r / g : INT32_MAX;
      const float sl2 = p.scale_log2;
      float m_used = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < nt; ++j, ++J) {
        const int b = J & 1, s = J & 1;
        mbar_wait(&bar_sfull[b], (J >> 1) & 1);
        tc_fence_after();
        float sv[N];
#pragma unroll
        for (int c = 0; c < N / 32; ++c) {
          float tmp[32];
          tmem_ld32(t_row + b * N + c * 32, tmp);
#pragma unroll
          for (int i = 0; i < 32; ++i) sv[c * 32 + i] = tmp[i];
        }
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bar_sfree[b]);
        const int key0 = it.k0 + j * N;
        const bool edge = (key0 + N > it.k1) || (key0 + N - 1 > pos);
        float mt = -CUDART_INF_F;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          float x = sv[i] * sl2;
          if (edge) {
            const int key = key0 + i;
            x = (key < it.k1 && key <= pos) ? x : -CUDART_INF_F;
          }
          sv[i] = x;
          mt = fmaxf(mt, x);
        }
        const float m_new = fmaxf(m_used, mt);
        float alpha = 1.f;
        bool rescale = false;
        if (m_new > m_used + 8.f) {  // lazy rescale (first tile: m_used = -inf)
          alpha = fast_exp2(m_used - m_new);
          m_used = m_new;
          rescale = true;
        }
        const float base = m_used == -CUDART_INF_F ? 0.f : m_used;
        float ps = 0.f;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          sv[i] = fast_exp2(sv[i] - base);
          ps += sv[i];
        }
        l = l * alpha + ps;
        if (j >= 1) mbar_wait(&bar_o, (J - 1) & 1);  // PV_{J-1} done: P free, O stable
        // tcgen05.ld/st are warp-collective: rescale the warp's rows if any of them needs it
        if (__any_sync(0xffffffffu, rescale) && j >= 1) {
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            float o[32];
            tmem_ld32(t_row + TM_O + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(t_row + TM_O + c * 32, o);
          }
          tmem_wait_st();
        }
        // P row (bf16) -> shared memory, K-major SW128 [key/64][row][64]
#pragma unroll
        for (int c = 0; c < N / 8; ++c) {
          uint4 v;
          v.x = pack_bf16(sv[c * 8 + 0], sv[c * 8 + 1]);
          v.y = pack_bf16(sv[c * 8 + 2], sv[c * 8 + 3]);
          v.z = pack_bf16(sv[c * 8 + 4], sv[c * 8 + 5]);
          v.w = pack_bf16(sv[c * 8 + 6], sv[c * 8 + 7]);
          *reinterpret_cast<uint4 *>(sP + kmaj_off(row, c * 8, M)) = v;
        }
        if (key0 + N > it.k1) {
          // last tile: zero V rows of keys >= k1 (NaN-poisoned / never loaded) before PV
          mbar_wait(&bar_fv[s], (J >> 1) & 1);
          const int vr = it.k1 - key0;
          const int nch = (N - vr) * HALVES * 8;
          for (int c = row; c < nch; c += 128) {
            const int key = vr + c / (HALVES * 8), rem = c % (HALVES * 8);
            const int h = rem >> 3, ch = rem & 7;
            *reinterpret_cast<uint4 *>(sV + s * TBYTES + h * (N * 128) + (key >> 3) * 1024 +
                                       (key & 7) * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(&bar_p);
      }
      // ------------------------------- epilogue -------------------------------
      mbar_wait(&bar_o, (J - 1) & 1);
      tc_fence_after();
      constexpr float kLn2 = 0.6931471805599453f;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -CUDART_INF_F;
      const int hq = it.kv_head * g + (valid ? r % g : 0);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        float o[32];
        tmem_ld32(t_row + TM_O + c * 32, o);
        tmem_wait_ld();
        if (!valid) continue;
        if (it.slot >= 0) {
          float4 *dst = reinterpret_cast<float4 *>(p.part_o + (int64_t)(it.slot + (r - it.r0)) * D + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(o[4 * i] * inv, o[4 * i + 1] * inv, o[4 * i + 2] * inv, o[4 * i + 3] * inv);
        } else if (p.out_f32) {
          float4 *dst = reinterpret_cast<float4 *>(reinterpret_cast<float *>(p.out) + (int64_t)qrow * p.o_stride_tok +
                                                   (int64_t)hq * p.o_stride_head + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dst[i] = make_float4(o[4 * i] * inv, o[4 * i + 1] * inv, o[4 * i + 2] * inv, o[4 * i + 3] * inv);
        } else {
          uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.out) + (int64_t)qrow * p.o_stride_tok +
                                                 (int64_t)hq * p.o_stride_head + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(o[8 * i] * inv, o[8 * i + 1] * inv), pack_bf16(o[8 * i + 2] * inv, o[8 * i + 3] * inv),
                                pack_bf16(o[8 * i + 4] * inv, o[8 * i + 5] * inv), pack_bf16(o[8 * i + 6] * inv, o[8 * i + 7] * inv));
        }
      }
      if (valid) {
        if (it.slot >= 0) p.part_lse[it.slot + (r - it.r0)] = lse;
        else if (p.lse) p.lse[(int64_t)qrow * p.Hq + hq] = lse;
      }
      tc_fence_before();  // O reads complete before the next item's first PV overwrites O
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int D>
static cudaError_t launch_tile_tc_t(const AttnParams &p, const void *tmk, const void *tmv,
                                    const TileItem *items, int n, int max_ctas, cudaStream_t s) {
  const size_t smem = (size_t)tc::M * D * 2 + 4 * (size_t)tc::N * D * 2 + (size_t)tc::M * tc::N * 2 + 1024;
  auto kern = tile_tc_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // full shared-memory carveout so CTAs of concurrently running kernels can share an SM
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::max(1, std::min(n, max_ctas > 0 ? max_ctas : nsm));
  kern<<<grid, 192, smem, s>>>(p, *reinterpret_cast<const CUtensorMap *>(tmk),
                               *reinterpret_cast<const CUtensorMap *>(tmv), items, n);
  return cudaGetLastError();
}

cudaError_t launch_tile_tc(const AttnParams &p, const void *tmk, const void *tmv,
                           const TileItem *items, int n, int max_ctas, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (p.d == 128) return launch_tile_tc_t<128>(p, tmk, tmv, items, n, max_ctas, s);
  return launch_tile_tc_t<64>(p, tmk, tmv, items, n, max_ctas, s);
}

}  // namespace kva
