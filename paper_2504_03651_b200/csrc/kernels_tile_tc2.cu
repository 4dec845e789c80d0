// kernels_tile_tc2.cu — tcgen05/TMEM tiled attention, two-Q-tile version (SURVEY §8(a) a3 +
// a5): prefill chunks ("compute-bound"; cost quadratic in length, Eq.(6)) and
// shared-prefix (cascade) tiles of the mixed batch.
//
// One persistent CTA processes work items of up to 256 query rows (r = tok*g + hh) as two
// 128-row Q tiles that SHARE every 128-key K/V tile (halving K/V traffic per flop):
//   warp 0      TMA producer: K and V rings, 2 stages each (2-D TMA, 128-B swizzle).
//   warp 1      TMEM allocator + MMA issuer (one elected lane):
//                 S_t = Q_t K_j^T   (SS: A=Q smem K-major, B=K smem K-major)  -> TMEM S_t
//                 O_t += P_t V_j     (TS: A=P in TMEM aliasing S_t, B=V smem MN-major) -> O_t
//               issue order per key tile j: QK0_j, PV1_{j-1}, QK1_j, PV0_j — the softmax of
//               one Q tile overlaps the MMAs of the other; S_t is rewritten only after the PV
//               that read P_t (in-order tcgen05 execution).
//   warps 2-5   softmax of Q tile 0, warps 6-9 softmax of Q tile 1: one thread per row
//               (= TMEM lane), tcgen05.ld of S, causal/range mask, online softmax in the
//               log2 domain with lazy O rescaling (only when the row max grows by > 8),
//               P (bf16) written back into TMEM with tcgen05.st; epilogue O/l from TMEM.
// TMEM columns: S0 [0,128), S1 [128,256), O0 [256,256+d), O1 [384,384+d).
#include <cuda.h>
#include <math_constants.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

namespace tc2 {

constexpr int M = 128;            // rows per Q tile (UMMA M, TMEM lanes)
constexpr int N = 128;            // keys per K/V tile
constexpr int NBLK = N / kBlock;  // 8 paged blocks per key tile
constexpr int THREADS = 320;      // 10 warps
#ifdef KVA_TILE_TIMESTAMPS
constexpr bool kTimestamps = true;
#else
constexpr bool kTimestamps = false;
#endif

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
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
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

// byte offset of element (row, col) in a K-major SW128 tile stored as [col/64][rows][64]
__device__ __forceinline__ uint32_t kmaj_off(int row, int col, int rows) {
  return (col >> 6) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
         ((((col & 63) >> 3) ^ (row & 7)) << 4) + ((col & 7) << 1);
}

struct ItemGeom {  // per-item derived quantities, identical in every role
  int kb0, nkb, nt, nt_t[2], rows_t[2], k1_t[2];
};
__device__ __forceinline__ ItemGeom geom(const TileItem &it, int g) {
  ItemGeom G;
  G.kb0 = it.k0 / kBlock;
  G.nkb = (it.k1 + kBlock - 1) / kBlock - G.kb0;
  G.nt = (G.nkb + NBLK - 1) / NBLK;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int rows = min(M, max(0, it.n_rows - t * M));
    G.rows_t[t] = rows;
    int k1 = it.k1;
    if (rows > 0 && (it.flags & kTileCausal)) k1 = min(it.k1, it.pos0 + (it.r0 + t * M + rows - 1) / g + 1);
    G.k1_t[t] = rows > 0 ? k1 : it.k0;
    G.nt_t[t] = rows > 0 ? (k1 - it.k0 + N - 1) / N : 0;
  }
  return G;
}

}  // namespace tc2

// PP = column pairs (of every 16) whose exp2 runs as a polynomial on the FMA pipe;
// V3 = V tiles loaded with one 3-D box per block-head (d = 128): V tile layout
// [block][half][16 keys][64] (PV reads it with LBO = 2 KB), else [half][128 keys][64]
template <int D, int PP, bool V3, bool K3>
__global__ void __launch_bounds__(tc2::THREADS, 1)
    tile_tc2_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const __grid_constant__ TileList L,
                    const __grid_constant__ CUtensorMap tmv3, const __grid_constant__ CUtensorMap tmk3) {
  const TileItem *items = L.ptr ? L.ptr : L.item;
  const int n_items = L.n;
  using namespace tc2;
  constexpr int HALVES = D / 64;
  constexpr int KBYTES = 16 * D * 2;  // one paged block, one head (K or V)
  constexpr int TBYTES = N * D * 2;   // one K or V tile
  constexpr int QBYTES = M * D * 2;   // one Q tile
  constexpr uint32_t ID_QK = idesc(M, N, false);
  constexpr uint32_t ID_PV = idesc(M, D, true);
  constexpr uint32_t COL_S[2] = {0, 128};
  constexpr uint32_t COL_O[2] = {256, 384};

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;                 // [2][QBYTES]
  uint8_t *sK = sQ + 2 * QBYTES;      // [2][TBYTES]
  uint8_t *sV = sK + 2 * TBYTES;      // [2][TBYTES]
  __shared__ uint64_t bar_q[2], bar_kf[2], bar_vf[2], bar_ke[2], bar_ve[2], bar_s[2], bar_p[2], bar_o[2];
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = p.g;
  // diagnostics: CTA 0 records %globaltimer at role events into p.dbg[role*512 + n]
  int dbg_n = 0;
  auto ts = [&](int role) {
#ifndef KVA_TILE_TIMESTAMPS  // role timelines (profiles/tc2_timeline.py) need -DKVA_TILE_TIMESTAMPS
    return;
#endif
    if (p.dbg && blockIdx.x == 0 && lane == 0 && dbg_n < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      p.dbg[role * 512 + dbg_n] = t;
    }
    ++dbg_n;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_q[i], 128);
      mbar_init(&bar_kf[i], 1);
      mbar_init(&bar_vf[i], 1);
      mbar_init(&bar_ke[i], 1);
      mbar_init(&bar_ve[i], 1);
      mbar_init(&bar_s[i], 1);
      mbar_init(&bar_p[i], 128);
      mbar_init(&bar_o[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base_s;
  // programmatic dependent launch: once every CTA of this persistent grid is resident, the
  // next kernel on the stream (the decode kernel, launched with the PDL attribute) may start
  // on the remaining SMs — the tile kernel claims its SMs first (it reads nothing the
  // dependent writes, and the dependent reads nothing this kernel writes)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.span && threadIdx.x == 0) {  // instrumentation: CTA start
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    atomicMin(&p.span[2], t0);
  }

  if (warp == 0) {
    // ------------------------------- TMA producer -------------------------------
    // launched as a dependent of the kv_append kernel: the rows it writes must be complete
    // (and visible) before the pool is read (a no-op for a normal launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int KT = 0;  // K/V tiles loaded so far (ring position)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const TileItem it = items[item];
      const ItemGeom G = geom(it, g);
      const int32_t *trow = p.block_table + (int64_t)it.table_row * p.max_blocks + G.kb0;
      for (int j = 0; j < G.nt; ++j, ++KT) {
        const int s = KT & 1;
        const int jb = j * NBLK + (lane & (NBLK - 1));
        const int id = (lane < NBLK && jb < G.nkb) ? __ldg(trow + jb) : 0;
        const int nb = min(NBLK, G.nkb - j * NBLK);
        int rows[NBLK];
#pragma unroll
        for (int q = 0; q < NBLK; ++q) rows[q] = (__shfl_sync(0xffffffffu, id, q) * p.Hkv + it.kv_head) * kBlock;
        if (KT >= 2) mbar_wait(&bar_ke[s], ((KT >> 1) - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bar_kf[s], nb * KBYTES);
          if constexpr (K3) {  // K tile [8-key group][half][8 keys][64]: one 4-D box per block
#pragma unroll
            for (int q = 0; q < NBLK; ++q)
              if (q < nb) tma_load_4d(sK + s * TBYTES + q * 4096, &tmk3, &bar_kf[s], 0, 0, 0, rows[q] >> 3);
          } else {
#pragma unroll
            for (int q = 0; q < NBLK; ++q)
              if (q < nb)
#pragma unroll
                for (int h = 0; h < HALVES; ++h)
                  tma_load_2d(sK + s * TBYTES + h * (N * 128) + q * 2048, &tmk, &bar_kf[s], h * 64, rows[q]);
          }
        }
        if (KT >= 2) mbar_wait(&bar_ve[s], ((KT >> 1) - 1) & 1);
        if (lane == 0) {
          mbar_arrive_expect_tx(&bar_vf[s], nb * KBYTES);
          if constexpr (V3) {
#pragma unroll
            for (int q = 0; q < NBLK; ++q)
              if (q < nb) tma_load_3d(sV + s * TBYTES + q * 4096, &tmv3, &bar_vf[s], 0, rows[q], 0);
          } else {
#pragma unroll
            for (int q = 0; q < NBLK; ++q)
              if (q < nb)
#pragma unroll
                for (int h = 0; h < HALVES; ++h)
                  tma_load_2d(sV + s * TBYTES + h * (N * 128) + q * 2048, &tmv, &bar_vf[s], h * 64, rows[q]);
          }
        }
        __syncwarp();
      }
    }
    // drain: observe the final release of every ring slot (keeps each mbarrier phase waited)
    for (int k = max(0, KT - 2); k < KT; ++k) {
      mbar_wait(&bar_ke[k & 1], (k >> 1) & 1);
      mbar_wait(&bar_ve[k & 1], (k >> 1) & 1);
    }
  } else if (warp == 1) {
    // ------------------------------- MMA issuer (whole warp loops, lane 0 issues) ------
    const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
    int KT0 = 0, Iq[2] = {0, 0}, Gp[2] = {0, 0};  // K/V tiles before this item, Q fills, PVs per tile-group
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const TileItem it = items[item];
      const ItemGeom G = geom(it, g);
      for (int t = 0; t < 2; ++t)
        if (G.rows_t[t] > 0) mbar_wait(&bar_q[t], Iq[t]++ & 1);
      fence_after();
      auto qk = [&](int t, int j) {  // S_t = Q_t K_j^T
        const int KT = KT0 + j, s = KT & 1;
        if (lane == 0) {
          if (!(p.debug_flags & 4)) {  // diagnostics: 4 = QK MMAs not issued (pipeline study)
            if constexpr (K3) {  // 8-key groups of a half are 2 KB apart: SBO = 2048, N = 128
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint64_t a = sdesc(q_base + t * QBYTES + (k >> 2) * (M * 128) + (k & 3) * 32, 16, 1024);
                const uint64_t b = sdesc(k_base + s * TBYTES + (k >> 2) * 1024 + (k & 3) * 32, 16, 2048);
                umma_ss(tmem + COL_S[t], a, b, ID_QK, k > 0 ? 1u : 0u);
              }
            } else {
#pragma unroll
              for (int k = 0; k < D / 16; ++k) {
                const uint64_t a = sdesc(q_base + t * QBYTES + (k >> 2) * (M * 128) + (k & 3) * 32, 16, 1024);
                const uint64_t b = sdesc(k_base + s * TBYTES + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024);
                umma_ss(tmem + COL_S[t], a, b, ID_QK, k > 0 ? 1u : 0u);
              }
            }
          }
          umma_commit(&bar_s[t]);
        }
        __syncwarp();
      };
      int vwaited = -1;
      auto pv = [&](int t, int j) {  // O_t += P_t V_j, P_t (bf16) in TMEM columns of S_t
        const int KT = KT0 + j, s = KT & 1;
        ts(0);
        mbar_wait(&bar_p[t], Gp[t] & 1);
        ts(0);
        if (vwaited != j) {
          mbar_wait(&bar_vf[s], (KT >> 1) & 1);
          vwaited = j;
          const int key0 = it.k0 + j * N;
          if (key0 + N > it.k1) {  // zero V rows of keys >= k1 (NaN-poisoned / never loaded)
            const int vr = it.k1 - key0;
            for (int c = lane; c < (N - vr) * HALVES * 8; c += 32) {
              const int key = vr + c / (HALVES * 8), rem = c % (HALVES * 8);
              const uint32_t off = V3 ? (uint32_t)((key >> 4) * 4096 + (rem >> 3) * 2048 + ((key >> 3) & 1) * 1024)
                                      : (uint32_t)((rem >> 3) * (N * 128) + (key >> 3) * 1024);
              *reinterpret_cast<uint4 *>(sV + s * TBYTES + off + (key & 7) * 128 + (rem & 7) * 16) =
                  make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async();
            __syncwarp();
          }
        }
        fence_after();
        if (lane == 0) {
          if (!(p.debug_flags & 2)) {  // diagnostics: 2 = PV MMAs not issued (pipeline study)
#pragma unroll
            for (int k = 0; k < N / 16; ++k) {
              const uint64_t b = V3 ? sdesc(v_base + s * TBYTES + k * 4096, 2048, 1024)
                                    : sdesc(v_base + s * TBYTES + k * 2048, N * 128, 1024);
              umma_ts(tmem + COL_O[t], tmem + COL_S[t] + k * 8, b, ID_PV, (j > 0 || k > 0) ? 1u : 0u);
            }
          }
          umma_commit(&bar_o[t]);
        }
        __syncwarp();
        ++Gp[t];
      };
      auto release = [&](uint64_t *bars, int j) {
        if (lane == 0) umma_commit(&bars[(KT0 + j) & 1]);
        __syncwarp();
      };
      const int nt0 = G.nt_t[0], nt1 = G.nt_t[1];
      for (int j = 0; j <= G.nt; ++j) {
        ts(0);
        if (j < G.nt) mbar_wait(&bar_kf[(KT0 + j) & 1], ((KT0 + j) >> 1) & 1);
        ts(0);
        if (j < nt0) qk(0, j);
        if (j >= 1 && j - 1 < nt1) {
          pv(1, j - 1);
          release(bar_ve, j - 1);        // PV0_{j-1} was issued before: V_{j-1} fully consumed
        }
        if (j < nt1) qk(1, j);
        if (j < G.nt) release(bar_ke, j);  // every QK of K_j issued
        if (j < nt0) {
          pv(0, j);
          if (j >= nt1) release(bar_ve, j);  // tile 1 does not use V_j
        }
      }
      KT0 += G.nt;
    }
  } else {
    // ------------------------------- softmax warp groups -------------------------------
    const int t = (warp - 2) >> 2;        // Q tile of this warp group
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane = row within the Q tile
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    uint8_t *sQt = sQ + t * QBYTES;
    int Gs = 0;  // S/P/O uses of this tile group (barrier phases)
    // Q_t of an item is staged by this warp group; the NEXT item's Q_t is staged right after
    // the last softmax step of the current one (its last QK_t has completed, so sQ_t is free),
    // before the epilogue: the MMA warp issues the next item's QKs while the epilogue drains O
    auto next_item = [&](int item) {  // next item with rows of this tile group
      for (; item < n_items; item += gridDim.x) {
        const TileItem it = items[item];
        const int n = it.n_rows - t * M;
        if (n > 0) break;
      }
      return item;
    };
    auto load_q = [&](int item) {  // stage Q_t of `item` into sQt; returns this row's q row
      const TileItem it = items[item];
      const int rows_t = min(M, it.n_rows - t * M);
      const int r = it.r0 + t * M + row;
      int qrow = 0;
      if (row < rows_t) {
        const int tok = r / g;
        qrow = (it.flags & kTileList) ? __ldg(p.row_list + it.row_src + tok) : it.row_src + tok;
        const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (int64_t)qrow * p.q_stride_tok +
                                                           (int64_t)(it.kv_head * g + r % g) * p.q_stride_head);
        uint4 v[D / 8];
#pragma unroll
        for (int c = 0; c < D / 8; ++c) v[c] = __ldg(src + c);
#pragma unroll
        for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4 *>(sQt + kmaj_off(row, c * 8, M)) = v[c];
      } else {
#pragma unroll
        for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4 *>(sQt + kmaj_off(row, c * 8, M)) = make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();
      mbar_arrive(&bar_q[t]);
      return qrow;
    };
    int item = next_item(blockIdx.x);
    int qrow_next = item < n_items ? load_q(item) : 0;
    for (; item < n_items;) {
      const TileItem it = items[item];
      const ItemGeom G = geom(it, g);
      const int rows_t = t ? G.rows_t[1] : G.rows_t[0];
      const int nt_t = t ? G.nt_t[1] : G.nt_t[0];
      const bool causal = it.flags & kTileCausal;
      const int r = it.r0 + t * M + row;
      const bool valid = row < rows_t;
      const int qrow = qrow_next;
      const int nxt = next_item(item + gridDim.x);
      const int pos = (causal && valid) ? it.pos0 + r / g : INT32_MAX;
      const int k1 = t ? G.k1_t[1] : G.k1_t[0];
      const float sl2 = p.scale_log2;
      float m_used = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < nt_t; ++j, ++Gs) {
        if (kTimestamps && (warp == 4 || warp == 8)) ts(1 + t);
        mbar_wait(&bar_s[t], Gs & 1);  // QK_t(j) done; so is PV_t(j-1) (issued earlier)
        if (j >= 1) mbar_wait(&bar_o[t], (Gs - 1) & 1);  // observe that completion (no-op wait)
        if (kTimestamps && (warp == 4 || warp == 8)) ts(1 + t);
        fence_after();
        if (p.debug_flags & 1) {  // diagnostics: measure the MMA/TMA pipeline without softmax
          fence_before();
          mbar_arrive(&bar_p[t]);
          continue;
        }
        // valid keys of this row in this tile: [key0, min(k1, pos + 1)) -> columns [0, lim)
        const int key0 = it.k0 + j * N;
        const int lim = max(0, min(min(k1, pos == INT32_MAX ? k1 : pos + 1) - key0, N));
        const bool full = __all_sync(0xffffffffu, lim == N);  // warp-uniform fast path
        auto load_all = [&](uint32_t (&u)[N]) {
#pragma unroll
          for (int c = 0; c < N / 32; ++c)
            ld32(t_row + COL_S[t] + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&u[c * 32]));
          wait_ld();
        };
        // pass 1: row max of the raw scores (scale > 0 commutes with max), 8 independent chains
        float mt;
        {
          uint32_t u[N];
          load_all(u);
          float m8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) m8[i] = -CUDART_INF_F;
          if (full) {  // 3-input max: half the instructions
#pragma unroll
            for (int i = 0; i < N; i += 2) m8[(i >> 1) & 7] = fmax3(m8[(i >> 1) & 7], __uint_as_float(u[i]), __uint_as_float(u[i + 1]));
          } else {
#pragma unroll
            for (int i = 0; i < N; ++i) m8[i & 7] = fmaxf(m8[i & 7], i < lim ? __uint_as_float(u[i]) : -CUDART_INF_F);
          }
          mt = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
          mt = mt == -CUDART_INF_F ? mt : mt * sl2;
        }
        const float m_new = fmaxf(m_used, mt);
        float alpha = 1.f;
        bool rescale = false;
        if (m_new > m_used + 8.f) {  // lazy rescale (first tile: m_used = -inf)
          alpha = fast_exp2(m_used - m_new);
          m_used = m_new;
          rescale = true;
        }
        const float nbase = m_used == -CUDART_INF_F ? 0.f : -m_used;
        // pass 2 (reload): P = exp2(s * scale - m), 4 independent row-sum chains, bf16 pairs
        // stored over S columns already read (P chunk c -> columns [16c, 16c+16))
        // paired fp32 ops (FFMA2/FADD2); kPolyPairs of every 16 column pairs take exp2 on the
        // FMA pipe (polynomial), the rest on MUFU, balancing the two units (PP of 16)
        float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc = make_float2(sl2, sl2), nb = make_float2(nbase, nbase);
#pragma unroll
        for (int hb = 0; hb < 2; ++hb) {  // 64-column halves: fewer live registers (no spills)
          uint32_t u[N];
#pragma unroll
          for (int c = 2 * hb; c < 2 * hb + 2; ++c)
            ld32(t_row + COL_S[t] + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&u[c * 32]));
          wait_ld();
          // two explicit copies of the loop: a warp-uniform branch instead of a per-element
          // compare + select that the compiler otherwise if-converts into every element
          auto exp_chunk = [&](int c, bool masked) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int i0 = c * 32 + 2 * i, i1 = i0 + 1;
              const float2 x = ffma2(make_float2(__uint_as_float(u[i0]), __uint_as_float(u[i1])), sc, nb);
              float2 e;
              if (i < PP) {
                e = exp2_poly2(x);
              } else {
                e.x = fast_exp2(x.x);
                e.y = fast_exp2(x.y);
              }
              if (masked) {
                e.x = i0 < lim ? e.x : 0.f;
                e.y = i1 < lim ? e.y : 0.f;
              }
              s2[i & 1] = fadd2(s2[i & 1], e);
              pk[i] = pack_bf16(e.x, e.y);
            }
            st16(t_row + COL_S[t] + c * 16, pk);
          };
          if (full) {
#pragma unroll
            for (int c = 2 * hb; c < 2 * hb + 2; ++c) exp_chunk(c, false);
          } else {
#pragma unroll
            for (int c = 2 * hb; c < 2 * hb + 2; ++c) exp_chunk(c, true);
          }
        }
        const float ps = (s2[0].x + s2[0].y) + (s2[1].x + s2[1].y);
        l = l * alpha + ps;
        if (__any_sync(0xffffffffu, rescale) && j >= 1) {  // warp-collective TMEM access
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            ld32(t_row + COL_O[t] + c * 32, o);
            wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            st32(t_row + COL_O[t] + c * 32, o);
          }
        }
        wait_st();
        fence_before();
        mbar_arrive(&bar_p[t]);
        if (kTimestamps && (warp == 4 || warp == 8)) ts(1 + t);
      }
      if (nxt < n_items) qrow_next = load_q(nxt);
      // ------------------------------- epilogue -------------------------------
      mbar_wait(&bar_o[t], (Gs - 1) & 1);
      fence_after();
      constexpr float kLn2 = 0.6931471805599453f;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const float lse = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -CUDART_INF_F;
      const int hq = it.kv_head * g + (valid ? r % g : 0);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t ou[32];
        ld32(t_row + COL_O[t] + c * 32, ou);
        wait_ld();
        if (!valid) continue;
        float o[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = __uint_as_float(ou[i]) * inv;
        if (it.slot >= 0) {
          float4 *dst = reinterpret_cast<float4 *>(p.part_o + (int64_t)(it.slot + (r - it.r0)) * D + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else {
          const int64_t off = (int64_t)qrow * p.o_stride_tok + (int64_t)hq * p.o_stride_head + c * 32;
          for (int oi = 0; oi <= p.n_out_extra; ++oi) {  // own output, then the peers' (fused a7)
            void *base = oi == 0 ? p.out : p.out_extra[oi - 1];
            if (p.out_f32) {
              float4 *dst = reinterpret_cast<float4 *>(reinterpret_cast<float *>(base) + off);
#pragma unroll
              for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
            } else {
              uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(base) + off);
#pragma unroll
              for (int i = 0; i < 4; ++i)
                dst[i] = make_uint4(pack_bf16(o[8 * i], o[8 * i + 1]), pack_bf16(o[8 * i + 2], o[8 * i + 3]),
                                    pack_bf16(o[8 * i + 4], o[8 * i + 5]), pack_bf16(o[8 * i + 6], o[8 * i + 7]));
            }
          }
        }
      }
      if (valid) {
        if (it.slot >= 0) p.part_lse[it.slot + (r - it.r0)] = lse;
        else if (p.lse) p.lse[(int64_t)qrow * p.Hq + hq] = lse;
      }
      if (p.fold_flags && (it.flags >> 8)) {  // a cascade item: this warp's partial rows are stored
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(p.fold_flags + 2 * ((it.flags >> 8) - 1) + t, 1u);
        }
      }
      fence_before();  // O reads done before this group's next item overwrites O
      item = nxt;
    }
  }
  fence_before();
  __syncthreads();
  if (p.span && threadIdx.x == 0) {  // instrumentation: CTA end (every role done)
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicMax(&p.span[3], t1);
  }
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int D, int PP, bool V3 = false, bool K3 = false>
static cudaError_t launch_tile_tc2_t(const AttnParams &p, const void *tmk, const void *tmv,
                                     const TileList &L, int max_ctas, cudaStream_t s, const void *tmv3,
                                     const void *tmk3 = nullptr) {
  const int n = L.n;
  const size_t smem = 2 * (size_t)tc2::M * D * 2 + 4 * (size_t)tc2::N * D * 2 + 1024;
  auto kern = tile_tc2_kernel<D, PP, V3, K3>;
  // max dynamic smem + full carveout (CTAs of concurrently running kernels share SMs), once
  cudaError_t e = smem_attrs_once(reinterpret_cast<const void *>(kern), (int)smem);
  if (e != cudaSuccess) return e;
  const int nsm = sm_count();
  const int grid = std::max(1, std::min(n, max_ctas > 0 ? max_ctas : nsm));
  // programmatic dependent launch: may become resident while the preceding kernel on the
  // stream (the kv_append of the tile-path rows) still runs; the producer waits for it
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(tc2::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, p, *reinterpret_cast<const CUtensorMap *>(tmk),
                            *reinterpret_cast<const CUtensorMap *>(tmv), L,
                            *reinterpret_cast<const CUtensorMap *>(V3 ? tmv3 : tmv),
                            *reinterpret_cast<const CUtensorMap *>(K3 ? tmk3 : tmk));
}

cudaError_t launch_tile_tc2(const AttnParams &p, const void *tmk, const void *tmv,
                            const TileList &items, int max_ctas, cudaStream_t s, const void *tmv3,
                            const void *tmk3) {
  if (items.n <= 0) return cudaSuccess;
  // the exp2 of the softmax stays on MUFU (round 1: moving 4 or 6 of 16 column pairs to an FMA-pipe
  // polynomial was slower, profiles/r01b/poly.log — this softmax is issue/latency-bound); K tiles by
  // one 4-D box per block and V by one 3-D box for d = 128 (llama70b 7.35 -> 7.21 ms vs 2-D boxes)
  if (p.d == 128) {
    if (!tmv3 || !tmk3) return cudaErrorInvalidValue;  // the pool always has them for d = 128
    return launch_tile_tc2_t<128, 0, true, true>(p, tmk, tmv, items, max_ctas, s, tmv3, tmk3);
  }
  return launch_tile_tc2_t<64, 0>(p, tmk, tmv, items, max_ctas, s, tmv3);
}

}  // namespace kva
