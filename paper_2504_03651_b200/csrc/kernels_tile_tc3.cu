// kernels_tile_tc3.cu — CTA-pair (tcgen05 cta_group::2) tiled attention for prefill chunks and
// shared-prefix tiles (SURVEY §8(a) a3 + a5), head_dim 128.
//
// Same algorithm as kernels_tile_tc2.cu (two Q slots per CTA, S/P/O in TMEM, interleaved
// QK0_j, PV1_{j-1}, QK1_j, PV0_j issue order, lazy O rescale), but every MMA is issued once
// for a CTA PAIR (cluster of 2 on one TPC) with M = 256: each CTA holds 128 rows of a slot
// (A operand and D in its own shared memory / TMEM) and HALF of the B operand — 64 keys of
// the K tile for S = Q K^T and 64 of the 128 V channels for O += P V.  Per SM this halves the
// K/V bytes loaded by TMA and cuts the tensor core's shared-memory operand traffic from
// 128 B/cycle (one-CTA SS-mode QK^T) to 96 B/cycle, the limit measured on tc2.
// A work item is 512 rows: slot t of CTA r holds rows [r0 + 256 t + 128 r, +128).
//
// Synchronisation (leader = cluster rank 0 issues every MMA):
//   * each CTA loads its K/V halves with local TMA (local full barriers); its warp 1 waits,
//     zeroes NaN/unloaded V rows of the last tile, and arrives on the LEADER's ready barrier
//     (count 2) — the leader MMA waits kready/vready;
//   * Q-ready / P-ready: each softmax warp (4 per slot per CTA) arrives on the leader's
//     barrier (count 8); the peer uses a cluster-scope remote arrive;
//   * MMA completion: tcgen05.commit multicast to both CTAs (S full, O done, ring empty).
#include <cuda.h>
#include <math_constants.h>

#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

namespace tc3 {

constexpr int M = 128;            // rows per CTA per slot (TMEM lanes)
constexpr int N = 128;            // keys per K/V tile
constexpr int NBLK = N / kBlock;  // 8 paged blocks per key tile
constexpr int D = 128;
constexpr int STAGES = 3;
constexpr int THREADS = 320;      // 10 warps

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void umma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// commit the issuing thread's prior MMAs to the barrier at this offset in BOTH CTAs
__device__ __forceinline__ void commit2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// address of the same shared-memory object in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa(const void *p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

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
__device__ __forceinline__ uint32_t kmaj_off(int row, int col, int rows) {
  return (col >> 6) * (rows * 128) + (row >> 3) * 1024 + (row & 7) * 128 +
         ((((col & 63) >> 3) ^ (row & 7)) << 4) + ((col & 7) << 1);
}

struct Geom {
  int kb0, nkb, nt, nt_t[2], rows_t[2], k1_t[2];
};
// item of up to 512 rows; slot t covers rows [256 t, 256 t + 256) of the item (both CTAs)
__device__ __forceinline__ Geom geom(const TileItem &it, int g) {
  Geom G;
  G.kb0 = it.k0 / kBlock;
  G.nkb = (it.k1 + kBlock - 1) / kBlock - G.kb0;
  G.nt = (G.nkb + NBLK - 1) / NBLK;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int rows = min(2 * M, max(0, it.n_rows - t * 2 * M));
    G.rows_t[t] = rows;
    int k1 = it.k1;
    if (rows > 0 && (it.flags & kTileCausal)) k1 = min(it.k1, it.pos0 + (it.r0 + t * 2 * M + rows - 1) / g + 1);
    G.k1_t[t] = rows > 0 ? k1 : it.k0;
    G.nt_t[t] = rows > 0 ? (k1 - it.k0 + N - 1) / N : 0;
  }
  return G;
}

}  // namespace tc3

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(tc3::THREADS, 1)
    tile_tc3_kernel(const AttnParams p, const __grid_constant__ CUtensorMap tmk,
                    const __grid_constant__ CUtensorMap tmv, const TileItem *__restrict__ items,
                    int n_items) {
  using namespace tc3;
  constexpr int KHALF = 64 * D * 2;       // 64 keys x 128 channels  (16 KB)
  constexpr int VHALF = N * 64 * 2;       // 128 keys x 64 channels  (16 KB)
  constexpr int QBYTES = M * D * 2;       // 32 KB per slot
  constexpr uint32_t ID_QK = idesc(2 * M, N, false);
  constexpr uint32_t ID_PV = idesc(2 * M, D, true);
  constexpr uint32_t COL_S[2] = {0, 128};
  constexpr uint32_t COL_O[2] = {256, 384};

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = smem;                       // [2][QBYTES]
  uint8_t *sK = sQ + 2 * QBYTES;            // [STAGES][KHALF]
  uint8_t *sV = sK + STAGES * KHALF;        // [STAGES][VHALF]
  __shared__ uint64_t bar_kf[STAGES], bar_vf[STAGES], bar_ke[STAGES], bar_ve[STAGES];
  __shared__ uint64_t bar_kr[STAGES], bar_vr[STAGES];  // leader: both halves ready (count 2)
  __shared__ uint64_t bar_q[2], bar_p[2];               // leader: count 8 warps (both CTAs)
  __shared__ uint64_t bar_s[2], bar_o[2];               // both CTAs: MMA commit multicast
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int g = p.g;
  int dbg_n = 0;
  auto ts = [&](int role) {  // diagnostics: CTA 0 role timelines into p.dbg (KVA_DEBUG_TS)
    if (p.dbg && blockIdx.x == 0 && lane == 0 && dbg_n < 512) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      p.dbg[role * 512 + dbg_n] = tt;
    }
    ++dbg_n;
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&bar_kf[i], 1);
      mbar_init(&bar_vf[i], 1);
      mbar_init(&bar_ke[i], 1);
      mbar_init(&bar_ve[i], 1);
      mbar_init(&bar_kr[i], 2);
      mbar_init(&bar_vr[i], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_q[i], 8);
      mbar_init(&bar_p[i], 8);
      mbar_init(&bar_s[i], 1);
      mbar_init(&bar_o[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  cluster_sync();  // barrier inits of both CTAs visible cluster-wide
  fence_after();
  const uint32_t tmem = tmem_base_s;

  if (warp == 0) {
    // ---------------------- TMA producer (both CTAs: own K/V halves) ----------------------
    int KT = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const TileItem it = items[item];
      const Geom G = geom(it, g);
      const int32_t *trow = p.block_table + (int64_t)it.table_row * p.max_blocks + G.kb0;
      for (int j = 0; j < G.nt; ++j, ++KT) {
        const int s = KT % STAGES, use = KT / STAGES;
        const int jb = j * NBLK + (lane & (NBLK - 1));
        const int id = (lane < NBLK && jb < G.nkb) ? __ldg(trow + jb) : 0;
        const int nb = min(NBLK, G.nkb - j * NBLK);
        int rows[NBLK];
#pragma unroll
        for (int q = 0; q < NBLK; ++q) rows[q] = (__shfl_sync(0xffffffffu, id, q) * p.Hkv + it.kv_head) * kBlock;
        ts(3);
        if (KT >= STAGES) mbar_wait(&bar_ke[s], (use - 1) & 1);  // K slot freed after the QKs
        ts(3);
        if (lane == 0) {
          // K: keys [64 rank, 64 rank + 64) of the tile = blocks 4 rank .. 4 rank + 3, all channels
          const int kq0 = 4 * (int)rank;
          const int nk = max(0, min(4, nb - kq0));
          mbar_arrive_expect_tx(&bar_kf[s], nk * 2 * 2048);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q < nk)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                tma_load_2d(sK + s * KHALF + h * (64 * 128) + q * 2048, &tmk, &bar_kf[s], h * 64, rows[kq0 + q]);
        }
        __syncwarp();
        if (KT >= STAGES) mbar_wait(&bar_ve[s], (use - 1) & 1);  // V slot freed after the PVs
        ts(3);
        if (lane == 0) {
          // V: all keys of the tile, channels [64 rank, 64 rank + 64)
          mbar_arrive_expect_tx(&bar_vf[s], nb * 2048);
#pragma unroll
          for (int q = 0; q < NBLK; ++q)
            if (q < nb) tma_load_2d(sV + s * VHALF + q * 2048, &tmv, &bar_vf[s], 64 * (int)rank, rows[q]);
        }
        __syncwarp();
      }
    }
    for (int k = max(0, KT - STAGES); k < KT; ++k) {  // observe the final releases
      mbar_wait(&bar_ke[k % STAGES], (k / STAGES) & 1);
      mbar_wait(&bar_ve[k % STAGES], (k / STAGES) & 1);
    }
  } else if (warp == 1) {
    // -------- warp 1: forward own K/V readiness to the leader; leader issues the MMAs --------
    const uint32_t q_base = smem_u32(sQ), k_base = smem_u32(sK), v_base = smem_u32(sV);
    int KT0 = 0, Iq[2] = {0, 0}, Gp[2] = {0, 0};
    for (int item = pair; item < n_items; item += npairs) {
      const TileItem it = items[item];
      const Geom G = geom(it, g);
      // readiness of tile j: wait own halves, zero own V rows >= k1, arrive on leader's barrier
      auto fwd_k = [&](int j) {
        const int KT = KT0 + j, s = KT % STAGES;
        mbar_wait(&bar_kf[s], (KT / STAGES) & 1);
        if (lane == 0) arrive_remote(mapa(&bar_kr[s], 0));
        __syncwarp();
      };
      auto fwd_v = [&](int j) {
        const int KT = KT0 + j, s = KT % STAGES;
        mbar_wait(&bar_vf[s], (KT / STAGES) & 1);
        const int key0 = it.k0 + j * N;
        if (key0 + N > it.k1) {
          const int vr = it.k1 - key0;
          for (int c = lane; c < (N - vr) * 8; c += 32) {
            const int key = vr + c / 8, ch = c % 8;
            *reinterpret_cast<uint4 *>(sV + s * VHALF + (key >> 3) * 1024 + (key & 7) * 128 + ch * 16) =
                make_uint4(0, 0, 0, 0);
          }
          fence_proxy_async();
          __syncwarp();
        }
        if (lane == 0) arrive_remote(mapa(&bar_vr[s], 0));
        __syncwarp();
      };
      if (!leader) {
        for (int j = 0; j < G.nt; ++j) {
          fwd_k(j);
          fwd_v(j);
        }
        KT0 += G.nt;
        continue;
      }
      for (int t = 0; t < 2; ++t)
        if (G.rows_t[t] > 0) mbar_wait(&bar_q[t], Iq[t]++ & 1);
      fence_after();
      auto qk = [&](int t, int j) {
        const int KT = KT0 + j, s = KT % STAGES;
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t a = sdesc(q_base + t * QBYTES + (k >> 2) * (M * 128) + (k & 3) * 32, 16, 1024);
            const uint64_t b = sdesc(k_base + s * KHALF + (k >> 2) * (64 * 128) + (k & 3) * 32, 16, 1024);
            umma2_ss(tmem + COL_S[t], a, b, ID_QK, k > 0 ? 1u : 0u);
          }
          commit2(&bar_s[t]);
        }
        __syncwarp();
      };
      auto pv = [&](int t, int j) {
        const int KT = KT0 + j, s = KT % STAGES;
        ts(0);
        mbar_wait(&bar_p[t], Gp[t] & 1);
        ts(0);
        fence_after();
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < N / 16; ++k) {
            const uint64_t b = sdesc(v_base + s * VHALF + k * 2048, 8192, 1024);
            umma2_ts(tmem + COL_O[t], tmem + COL_S[t] + k * 8, b, ID_PV, (j > 0 || k > 0) ? 1u : 0u);
          }
          commit2(&bar_o[t]);
        }
        __syncwarp();
        ++Gp[t];
      };
      auto release = [&](uint64_t *bars, int j) {
        if (lane == 0) commit2(&bars[(KT0 + j) % STAGES]);
        __syncwarp();
      };
      const int nt0 = G.nt_t[0], nt1 = G.nt_t[1];
      int vready = -1;
      auto ensure_v = [&](int j) {
        if (vready >= j) return;
        fwd_v(j);  // own half (leader) -> arrival on own bar_vr
        const int KT = KT0 + j, s = KT % STAGES;
        ts(0);
        mbar_wait(&bar_vr[s], (KT / STAGES) & 1);
        ts(0);
        vready = j;
      };
      for (int j = 0; j <= G.nt; ++j) {
        ts(0);
        if (j < G.nt) {
          fwd_k(j);
          ts(0);
          const int KT = KT0 + j;
          mbar_wait(&bar_kr[KT % STAGES], (KT / STAGES) & 1);
          ts(0);
          fence_after();
        }
        if (j < nt0) qk(0, j);
        if (j >= 1 && j - 1 < nt1) {
          ensure_v(j - 1);
          pv(1, j - 1);
          release(bar_ve, j - 1);
        }
        if (j < nt1) qk(1, j);
        if (j < G.nt) release(bar_ke, j);
        if (j < nt0) {
          ensure_v(j);
          pv(0, j);
          if (j >= nt1) release(bar_ve, j);
        }
      }
      KT0 += G.nt;
    }
  } else {
    // ------------------------------- softmax warp groups -------------------------------
    const int t = (warp - 2) >> 2;        // slot of this warp group
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;  // TMEM lane = row within this CTA's half of the slot
    const uint32_t t_row = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t bar_q_l = mapa(&bar_q[t], 0), bar_p_l = mapa(&bar_p[t], 0);
    uint8_t *sQt = sQ + t * QBYTES;
    int Gs = 0;
    for (int item = pair; item < n_items; item += npairs) {
      const TileItem it = items[item];
      const Geom G = geom(it, g);
      if (G.rows_t[t] == 0) continue;
      const bool is_list = it.flags & kTileList, causal = it.flags & kTileCausal;
      const int lr = t * 2 * M + (int)rank * M + row;  // row index within the item
      const int r = it.r0 + lr;
      const bool valid = lr < it.n_rows;
      int qrow = 0;
      if (valid) {
        const int tok = r / g;
        qrow = is_list ? __ldg(p.row_list + it.row_src + tok) : it.row_src + tok;
        const uint4 *src = reinterpret_cast<const uint4 *>(p.q + (int64_t)qrow * p.q_stride_tok +
                                                           (int64_t)(it.kv_head * g + r % g) * p.q_stride_head);
#pragma unroll
        for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4 *>(sQt + kmaj_off(row, c * 8, M)) = __ldg(src + c);
      } else {
#pragma unroll
        for (int c = 0; c < D / 8; ++c) *reinterpret_cast<uint4 *>(sQt + kmaj_off(row, c * 8, M)) = make_uint4(0, 0, 0, 0);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) arrive_remote(bar_q_l);

      const int pos = (causal && valid) ? it.pos0 + r / g : INT32_MAX;
      const int k1 = G.k1_t[t];
      const float sl2 = p.scale_log2;
      float m_used = -CUDART_INF_F, l = 0.f;
      for (int j = 0; j < G.nt_t[t]; ++j, ++Gs) {
        if (warp == 4 || warp == 8) ts(1 + t);
        mbar_wait(&bar_s[t], Gs & 1);
        if (j >= 1) mbar_wait(&bar_o[t], (Gs - 1) & 1);
        if (warp == 4 || warp == 8) ts(1 + t);
        fence_after();
        const int key0 = it.k0 + j * N;
        const int lim = max(0, min(min(k1, pos == INT32_MAX ? k1 : pos + 1) - key0, N));
        const bool full = __all_sync(0xffffffffu, lim == N);
        auto load_all = [&](uint32_t (&u)[N]) {
#pragma unroll
          for (int c = 0; c < N / 32; ++c)
            ld32(t_row + COL_S[t] + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&u[c * 32]));
          wait_ld();
        };
        float mt;
        {
          uint32_t u[N];
          load_all(u);
          float m8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) m8[i] = -CUDART_INF_F;
          if (full) {
#pragma unroll
            for (int i = 0; i < N; ++i) m8[i & 7] = fmaxf(m8[i & 7], __uint_as_float(u[i]));
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
        if (m_new > m_used + 8.f) {
          alpha = fast_exp2(m_used - m_new);
          m_used = m_new;
          rescale = true;
        }
        const float nbase = m_used == -CUDART_INF_F ? 0.f : -m_used;
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
        {
          uint32_t u[N];
          load_all(u);
#pragma unroll
          for (int c = 0; c < N / 32; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int i0 = c * 32 + 2 * i, i1 = i0 + 1;
              float e0 = fast_exp2(fmaf(__uint_as_float(u[i0]), sl2, nbase));
              float e1 = fast_exp2(fmaf(__uint_as_float(u[i1]), sl2, nbase));
              if (!full) {
                e0 = i0 < lim ? e0 : 0.f;
                e1 = i1 < lim ? e1 : 0.f;
              }
              s4[i & 3] += e0 + e1;
              pk[i] = pack_bf16(e0, e1);
            }
            st16(t_row + COL_S[t] + c * 16, pk);
          }
        }
        l = l * alpha + ((s4[0] + s4[1]) + (s4[2] + s4[3]));
        if (__any_sync(0xffffffffu, rescale) && j >= 1) {
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
        __syncwarp();
        if (lane == 0) arrive_remote(bar_p_l);
        if (warp == 4 || warp == 8) ts(1 + t);
      }
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
          float4 *dst = reinterpret_cast<float4 *>(p.part_o + (int64_t)(it.slot + lr) * D + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else if (p.out_f32) {
          float4 *dst = reinterpret_cast<float4 *>(reinterpret_cast<float *>(p.out) + (int64_t)qrow * p.o_stride_tok +
                                                   (int64_t)hq * p.o_stride_head + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
        } else {
          uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<uint16_t *>(p.out) + (int64_t)qrow * p.o_stride_tok +
                                                 (int64_t)hq * p.o_stride_head + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(o[8 * i], o[8 * i + 1]), pack_bf16(o[8 * i + 2], o[8 * i + 3]),
                                pack_bf16(o[8 * i + 4], o[8 * i + 5]), pack_bf16(o[8 * i + 6], o[8 * i + 7]));
        }
      }
      if (valid) {
        if (it.slot >= 0) p.part_lse[it.slot + lr] = lse;
        else if (p.lse) p.lse[(int64_t)qrow * p.Hq + hq] = lse;
      }
      fence_before();
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs done with every MMA and TMEM access
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

cudaError_t launch_tile_tc3(const AttnParams &p, const void *tmk, const void *tmv,
                            const TileItem *items, int n, int max_ctas, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = 2 * (size_t)tc3::M * tc3::D * 2 + tc3::STAGES * (size_t)(64 * tc3::D * 2 + tc3::N * 64 * 2) + 1024;
  cudaError_t e = cudaFuncSetAttribute(tile_tc3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(tile_tc3_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = std::max(2, std::min(2 * n, max_ctas > 0 ? max_ctas : nsm)) & ~1;
  tile_tc3_kernel<<<ctas, tc3::THREADS, smem, s>>>(p, *reinterpret_cast<const CUtensorMap *>(tmk),
                                                   *reinterpret_cast<const CUtensorMap *>(tmv), items, n);
  return cudaGetLastError();
}

}  // namespace kva
