// kernels_select.cuh — evict_select: the first k blocks of the eviction order.
// Compiled twice: kernels_select.cu (512 threads per CTA, 2,048-pair CTA buckets: the fastest
// alone) and kernels_select256.cu (256 threads, 1,024-pair buckets, ~30 KB of shared memory:
// shares its SM with two decode CTAs); option evict_threads picks one per call.
//
// Order: "When evicting the KV cache, we will first consider the priority of the KV cache
// entry, and then the last access time" (priorities P:331-334, encoded into the u64
// keys by evict_keys, readings #18-#20); equal keys are broken by block id.  The result
// is the ascending (key, id) order of the evictable keys (key != UINT64_MAX), truncated to k
// ("victims ... in eviction order").
//
// One cooperative persistent kernel (C CTAs x 512 threads, grid barriers between phases) runs
// a most-significant-digit radix partition truncated to the top k, on a "composite" key that
// is unique per block: the bits that vary among the evictable keys (constant bits carry no
// order), followed by the block id.  Composite order == (key, id) order.
//   phase 0   OR / OR-of-complements / count of the evictable keys (-> which bits vary, E)
//   phase 1   histogram of the top 11-bit digit; each CTA reserves its range in every bin
//   round r   every CTA scans the digit-r histogram, finds the boundary bin b holding rank
//             k-1 of the current segment, and scatters its elements: bins < b are taken
//             (their output range is known: bin start = exclusive prefix), bin b is either
//             taken whole, finished by one sort (<= kCap elements) or becomes the next
//             round's segment (its digit r+1 is counted in the same pass), bins > b dropped
//   buckets   every taken bin with >= 2 elements is a bucket at a known output offset: warps
//             sort buckets of <= 256 pairs in registers, CTAs sort <= 2048 (registers +
//             shared-memory exchanges), larger ones are partitioned again by one CTA (next
//             digit) -> next level
// The k-th element's bin shrinks ~2048x per round, so the uniform-ish `evict` workload needs
// two rounds over 2^20 and ~125k keys, and one bucket level: four grid barriers in all.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "internal.h"

namespace cg = cooperative_groups;

namespace kva {
namespace {

#ifndef KVA_SEL_THREADS
#define KVA_SEL_THREADS 512
#endif
#ifndef KVA_SEL_VARIANT
#define KVA_SEL_VARIANT 512
#endif
#define KVA_SEL_CAT2(a, b) a##b
#define KVA_SEL_CAT(a, b) KVA_SEL_CAT2(a, b)
constexpr int kT = KVA_SEL_THREADS;  // threads per CTA
constexpr int kNW = kT / 32;
#ifndef KVA_SEL_DIGIT
#define KVA_SEL_DIGIT 11
#endif
constexpr int kDig = KVA_SEL_DIGIT;  // radix digit bits
constexpr int kBins = 1 << kDig;
constexpr int kPer = kBins / kT;      // histogram bins per thread in the scans
#ifndef KVA_SEL_CAP
#define KVA_SEL_CAP 2048
#endif
constexpr int kCap = KVA_SEL_CAP;    // pairs one CTA sorts in shared memory (24 KB at 2048)
constexpr int kWarpMax = 256;        // pairs one warp sorts in registers (8 per lane)
constexpr int kMaxRuns = 8;          // runs of varying key bits kept apart (more are merged)
constexpr int kMaxLevels = 16;
constexpr int kMaxC = 512;
constexpr uint64_t kInf = ~0ull;

struct Part {  // per-CTA phase-0 result
  unsigned long long o, a, c, pad;
};
struct Ctl {
  unsigned long long t[32];  // phase timestamps of CTA 0 (%globaltimer ns; diagnostics)
  unsigned int n_small[kMaxLevels], n_large[kMaxLevels], n_big[kMaxLevels];
  unsigned int rounds, levels, pad[2];
  unsigned long long v_prev;  // the varying-bit mask of the last call on this workspace
};

struct Layout {
  size_t ctl, part, hist, wk[2], wi[2], sk[2], si[2], rs[2], rl[2], total;
  int64_t nw, ns, nrec;
};
inline size_t up256(size_t x) { return (x + 255) & ~size_t(255); }
Layout layout(int64_t n, int64_t k) {
  Layout L{};
  L.nw = std::max<int64_t>(n, 1);
  L.ns = std::min<int64_t>(std::max<int64_t>(k, 1), L.nw) + kCap;
  L.nrec = L.ns / 2 + 64;
  size_t p = 0;
  auto take = [&](size_t bytes) { const size_t at = p; p = up256(p + bytes); return at; };
  L.ctl = take(sizeof(Ctl));
  L.part = take(sizeof(Part) * kMaxC);
  L.hist = take(sizeof(unsigned int) * 3 * kBins);
  for (int i = 0; i < 2; ++i) L.wk[i] = take(8 * (size_t)L.nw);
  for (int i = 0; i < 2; ++i) L.wi[i] = take(4 * (size_t)L.nw);
  for (int i = 0; i < 2; ++i) L.sk[i] = take(8 * (size_t)L.ns);
  for (int i = 0; i < 2; ++i) L.si[i] = take(4 * (size_t)L.ns);
  for (int i = 0; i < 2; ++i) L.rs[i] = take(16 * (size_t)L.nrec);
  for (int i = 0; i < 2; ++i) L.rl[i] = take(16 * (size_t)L.nrec);
  L.total = p;
  return L;
}

struct SelArgs {
  const uint64_t *keys;
  int64_t n, k;
  int32_t *out_ids;
  int64_t *d_count;
  uint32_t *free_bits;  // nullable: apply (mark the selected blocks free)
  Ctl *ctl;
  Part *part;
  unsigned int *hist;  // [3][kBins]
  uint64_t *wk[2];     // segment (key, id) ping-pong, [n]
  int32_t *wi[2];
  uint64_t *sk[2];     // output-aligned staging ping-pong, [k + kCap]
  int32_t *si[2];
  uint4 *rs[2], *rl[2];  // bucket records (off, size, take, dig | src << 8): <= 256 / larger
  unsigned long long *span;  // diagnostics (span_ring): {CTA 0 start, latest CTA end}
  int fused;                 // the manager step runs first (mgr; its keys pass is phase 0's input)
  MgrArgs mgr;
};

__device__ __forceinline__ bool pair_gt(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
  return ka > kb || (ka == kb && ia > ib);
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan (kT threads); `total` = block sum.  Ends with a barrier.
__device__ __forceinline__ unsigned block_scan(unsigned v, unsigned *s_w, unsigned &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    unsigned t = lane < kNW ? s_w[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kNW) s_w[lane] = t;
  }
  __syncthreads();
  total = s_w[kNW - 1];
  const unsigned r = x - v + (w > 0 ? s_w[w - 1] : 0u);
  __syncthreads();
  return r;
}

// Shared-memory histogram increment (d < 0: none).  The lanes sharing the first valid lane's
// digit (the common case: neighbouring blocks of one chain share their class) are counted by
// one atomic, the others one by one.
__device__ __forceinline__ void hist_add(unsigned *h, int d) {
  const unsigned valid = __ballot_sync(0xffffffffu, d >= 0);
  if (!valid) return;
  const int leader = __ffs(valid) - 1;
  const int d0 = __shfl_sync(0xffffffffu, d, leader);
  const unsigned same = __ballot_sync(0xffffffffu, d == d0);
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(&h[d0], (unsigned)__popc(same));
  else if (d >= 0 && d != d0) atomicAdd(&h[d], 1u);
}

// Position of this lane's element in bin d (d < 0: none): the pre-increment value of cur[d]
// plus its rank among the lanes that share the first valid lane's digit (one atomic for them).
__device__ __forceinline__ unsigned bin_claim(unsigned *cur, int d) {
  const unsigned valid = __ballot_sync(0xffffffffu, d >= 0);
  if (!valid) return 0u;
  const int leader = __ffs(valid) - 1;
  const int d0 = __shfl_sync(0xffffffffu, d, leader);
  const unsigned same = __ballot_sync(0xffffffffu, d == d0);
  unsigned base = 0;
  if ((int)(threadIdx.x & 31) == leader) base = atomicAdd(&cur[d0], (unsigned)__popc(same));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (d == d0) return base + __popc(same & lanemask_lt());
  return d >= 0 ? atomicAdd(&cur[d], 1u) : 0u;
}

// Batched forms for NK keys per lane (the input passes): the lanes' keys that share the
// warp's dominant digit (the first valid one; neighbouring blocks of a chain share their
// class and LAT) are counted / claimed with ONE shared atomic for all NK keys — the hot bin
// otherwise takes one same-address atomic per warp per key, serialised across the CTA's warps.
template <int NK>
__device__ __forceinline__ int dominant(const int (&d)[NK]) {
  int D = -1;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    const unsigned v = __ballot_sync(0xffffffffu, d[k] >= 0);
    if (D < 0 && v) D = __shfl_sync(0xffffffffu, d[k], __ffs(v) - 1);
  }
  return D;
}
template <int NK>
__device__ __forceinline__ void hist_batch(unsigned *h, const int (&d)[NK]) {
  const int D = dominant(d);
  if (D < 0) return;
  unsigned tot = 0;
#pragma unroll
  for (int k = 0; k < NK; ++k) tot += __popc(__ballot_sync(0xffffffffu, d[k] == D));
  if ((threadIdx.x & 31) == 0) atomicAdd(&h[D], tot);
#pragma unroll
  for (int k = 0; k < NK; ++k)
    if (d[k] >= 0 && d[k] != D) atomicAdd(&h[d[k]], 1u);
}
template <int NK>
__device__ __forceinline__ void claim_batch(unsigned *cur, const int (&d)[NK], unsigned (&pos)[NK]) {
  const int D = dominant(d);
  if (D < 0) return;
  unsigned same[NK], tot = 0;
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    same[k] = __ballot_sync(0xffffffffu, d[k] == D);
    tot += __popc(same[k]);
  }
  unsigned base = 0;
  if ((threadIdx.x & 31) == 0) base = atomicAdd(&cur[D], tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < NK; ++k) {
    if (d[k] == D) pos[k] = base + __popc(same[k] & lt);
    base += __popc(same[k]);
  }
#pragma unroll
  for (int k = 0; k < NK; ++k)
    if (d[k] >= 0 && d[k] != D) pos[k] = atomicAdd(&cur[d[k]], 1u);
}

// Add this CTA's bin counts to the grid's (global) counts; s_off[d] = this CTA's offset in bin d.
// The kBins / kT atomics of a thread are issued before any result is used (L2 round trips).
__device__ __forceinline__ void flush_counts(const unsigned *s_cnt, unsigned *s_off, unsigned *g) {
  constexpr int U = kBins / kT;
  unsigned v[U], o[U];
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = s_cnt[threadIdx.x + u * kT];
#pragma unroll
  for (int u = 0; u < U; ++u) o[u] = v[u] ? atomicAdd(&g[threadIdx.x + u * kT], v[u]) : 0u;
#pragma unroll
  for (int u = 0; u < U; ++u) s_off[threadIdx.x + u * kT] = o[u];
}

// The composite key: the compressed key ck (the varying key bits, runs packed towards bit 0,
// most significant run highest: ck = sum_i (key & mask_i) >> sh_i, an order-preserving
// injection on the evictable keys), then idb id bits.  Segments, staging and buckets hold
// (ck, id); only the input keys are compressed (once per pass over them).
struct Comp {
  unsigned long long v;  // the varying-bit mask it was made for
  int nr, idb, B, nd;
  unsigned long long cst;  // the key bits outside the runs (equal in every evictable key)
  unsigned long long mask[kMaxRuns];
  int sh[kMaxRuns];
  // digit 0 straight from the raw key when it lies within the key bits (n0 >= 0): the sum of
  // (key & m0[i]) >> s0[i] over the n0 runs that reach into its window; n0 < 0: via compress
  int n0;
  unsigned long long m0[kMaxRuns];
  int s0[kMaxRuns];
};
// The composite layout for varying-bit mask V (cst is set by the caller): runs of V, most
// significant first, gaps merged (smallest first) past kMaxRuns; any V gives a valid layout
// for keys whose varying bits lie inside it.
__device__ void make_comp(Comp &out, uint64_t V, int64_t n) {
  // run i = bits [rlo[i], rhi[i]] (i = 0 most significant): the i-th highest of the runs'
  // top bits (V & ~(V >> 1)) and bottom bits (V & ~(V << 1)); registers in the common case
  int rlo[kMaxRuns], rhi[kMaxRuns];
  int nr = __popcll(V & ~(V << 1));
  if (nr <= kMaxRuns) {
    uint64_t hs = V & ~(V >> 1), ls = V & ~(V << 1);
#pragma unroll
    for (int i = 0; i < kMaxRuns; ++i) {
      rhi[i] = hs ? 63 - __clzll((long long)hs) : 0;
      rlo[i] = ls ? 63 - __clzll((long long)ls) : 0;
      if (hs) { hs &= ~(1ull << rhi[i]); ls &= ~(1ull << rlo[i]); }
    }
  } else {  // more runs than kept apart: merge the smallest gaps
    int xl[32], xh[32], m = 0;
    for (uint64_t rem = V; rem;) {
      const int hb = 63 - __clzll((long long)rem);
      const uint64_t zeros = hb ? (~rem & ((1ull << hb) - 1ull)) : 0ull;  // clear bits below hb
      const int lb = zeros ? 64 - __clzll((long long)zeros) : 0;            // run = [lb, hb]
      xh[m] = hb; xl[m] = lb; ++m;
      rem &= lb ? ((1ull << lb) - 1ull) : 0ull;
    }
    while (m > kMaxRuns) {
      int best = 0, gap = 1 << 30;
      for (int i = 0; i + 1 < m; ++i) {
        const int g = xl[i] - xh[i + 1];
        if (g < gap) { gap = g; best = i; }
      }
      xl[best] = xl[best + 1];
      for (int i = best + 1; i + 1 < m; ++i) { xl[i] = xl[i + 1]; xh[i] = xh[i + 1]; }
      --m;
    }
    nr = m;
#pragma unroll
    for (int i = 0; i < kMaxRuns; ++i) { rlo[i] = xl[i]; rhi[i] = xh[i]; }
  }
  out.v = V;
  out.nr = nr;
  out.cst = 0ull;
  int bits = 0;
#pragma unroll
  for (int i = kMaxRuns - 1; i >= 0; --i) {  // least significant run lands at bit 0
    const int len = rhi[i] - rlo[i] + 1;
    out.mask[i] = i < nr ? (len >= 64 ? ~0ull : ((1ull << len) - 1ull)) << rlo[i] : 0ull;
    out.sh[i] = i < nr ? rlo[i] - bits : 0;
    bits += i < nr ? len : 0;
    out.m0[i] = 0ull;
    out.s0[i] = 0;
  }
  const int idb = n <= 1 ? 0 : min(31, 64 - __clzll((long long)(n - 1)));
  out.idb = idb;
  const int B = bits + idb;
  out.B = B;
  out.nd = B > 0 ? (B + kDig - 1) / kDig : 1;
  // digit-0 window [lo0, B) of the composite -> [wl, wh) of the compressed key
  const int lo0 = B > kDig ? B - kDig : 0;
  int n0 = -1;
  if (lo0 >= idb) {
    const int wl = lo0 - idb, wh = B - idb;
    n0 = 0;
#pragma unroll
    for (int i = 0; i < kMaxRuns; ++i) {  // run i: key bit j -> compressed bit j - sh[i]
      if (i >= nr) break;
      const int jl = wl + out.sh[i], jh = wh + out.sh[i];  // key bits [jl, jh) land in the window
      if (jl >= 64) continue;
      const uint64_t win = (jh >= 64 ? ~0ull : ((1ull << jh) - 1ull)) & ~((1ull << jl) - 1ull);
      if (out.mask[i] & win) {
        out.m0[n0] = out.mask[i] & win;
        out.s0[n0] = jl;
        ++n0;
      }
    }
  }
  out.n0 = n0;
}

// the first 4 runs in registers (the `evict` keys have 3: priority code, LAT, depth), the
// rest read from shared memory
struct CompR {
  int nr;
  unsigned long long m0, m1, m2, m3;
  int s0, s1, s2, s3;
  const Comp *c;
};
// digit 0 from the raw key (Comp::n0 >= 0): the first two contributing runs in registers
struct Dig0R {
  int n0;
  unsigned long long m0, m1;
  int s0, s1;
  const Comp *c;
};
__device__ __forceinline__ Dig0R dig0_regs(const Comp &c) {
  Dig0R r;
  r.n0 = c.n0;
  r.m0 = c.m0[0]; r.m1 = c.n0 > 1 ? c.m0[1] : 0ull;
  r.s0 = c.s0[0]; r.s1 = c.n0 > 1 ? c.s0[1] : 0;
  r.c = &c;
  return r;
}
__device__ __forceinline__ int digit0_raw(const Dig0R &r, uint64_t key) {
  uint32_t d = (uint32_t)((key & r.m0) >> r.s0) | (uint32_t)((key & r.m1) >> r.s1);
  if (r.n0 > 2)
    for (int i = 2; i < r.n0; ++i) d |= (uint32_t)((key & r.c->m0[i]) >> r.c->s0[i]);
  return (int)d;
}
__device__ __forceinline__ CompR comp_regs(const Comp &c) {
  CompR r;
  r.nr = c.nr;
  r.m0 = c.mask[0]; r.m1 = c.mask[1]; r.m2 = c.mask[2]; r.m3 = c.mask[3];
  r.s0 = c.sh[0]; r.s1 = c.sh[1]; r.s2 = c.sh[2]; r.s3 = c.sh[3];
  r.c = &c;
  return r;
}
__device__ __forceinline__ uint64_t compress(const CompR &r, uint64_t key) {
  uint64_t ck = ((key & r.m0) >> r.s0) | ((key & r.m1) >> r.s1) | ((key & r.m2) >> r.s2) | ((key & r.m3) >> r.s3);
  if (r.nr > 4)
    for (int i = 4; i < r.nr; ++i) ck |= (key & r.c->mask[i]) >> r.c->sh[i];
  return ck;
}
// bits [lo, lo + w) of the composite (ck << idb) | id, w <= kDig
struct DigSel {
  int lo, w, idb;
};
__device__ __forceinline__ DigSel dig_sel(const Comp &c, int r) {
  const int hi = c.B - kDig * r;
  DigSel d;
  d.lo = hi > kDig ? hi - kDig : 0;
  d.w = hi > d.lo ? hi - d.lo : 0;
  d.idb = c.idb;
  return d;
}
__device__ __forceinline__ int digit(const DigSel &s, uint64_t ck, int32_t id) {
  uint64_t v;
  if (s.lo >= s.idb) v = ck >> (s.lo - s.idb);
  else v = (ck << (s.idb - s.lo)) | ((uint64_t)(uint32_t)id >> s.lo);  // idb - lo <= kDig
  return (int)((uint32_t)v & ((1u << s.w) - 1u));
}

__device__ __forceinline__ void emit(const SelArgs &a, int64_t pos, int32_t id) {
  a.out_ids[pos] = id;
  if (a.free_bits) atomicOr(a.free_bits + (id >> 5), 1u << (id & 31));
}

// Bitonic sort of N = G*E pairs held by a group of G threads (G = 32: one warp; G = kT: the
// CTA), element j of thread t = index G*j + t.  Exchanges at stride >= G stay in the thread,
// 32 <= stride < G go through shared memory (sbk / sbi, G*E pairs), stride < 32 by shuffles.
// Stage loops are not unrolled (instruction-cache footprint).
template <int E, int G>
__device__ __forceinline__ void group_sort(uint64_t (&x)[E], int32_t (&y)[E], uint64_t *sbk, int32_t *sbi) {
  const int t = G == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  constexpr unsigned N = (unsigned)G * E;
#pragma unroll 1
  for (unsigned s2 = 2; s2 <= N; s2 <<= 1) {
#pragma unroll 1
    for (unsigned st = s2 >> 1; st > 0; st >>= 1) {
      if (st >= (unsigned)G) {
        const unsigned js = st / G;  // 1, 2 or 4 (E <= 8)
        auto pass = [&](auto jsc) {
          constexpr int JS = decltype(jsc)::value;
#pragma unroll
          for (int j = 0; j < E; ++j) {
            if ((j & JS) || (j | JS) >= E) continue;
            const int k = j | JS;
            const bool asc = (((unsigned)(G * j + t)) & s2) == 0;
            if (pair_gt(x[j], y[j], x[k], y[k]) == asc) {
              const uint64_t tk = x[j]; x[j] = x[k]; x[k] = tk;
              const int32_t ti = y[j]; y[j] = y[k]; y[k] = ti;
            }
          }
        };
        if (js == 1) pass(std::integral_constant<int, 1>{});
        else if (js == 2) pass(std::integral_constant<int, 2>{});
        else pass(std::integral_constant<int, 4>{});
      } else if (st >= 32) {
#pragma unroll
        for (int j = 0; j < E; ++j) { sbk[G * j + t] = x[j]; sbi[G * j + t] = y[j]; }
        __syncthreads();
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const unsigned i = (unsigned)(G * j + t), p = i ^ st;
          const uint64_t px = sbk[p];
          const int32_t py = sbi[p];
          const bool keep_min = ((i & st) == 0) == ((i & s2) == 0);
          if (pair_gt(x[j], y[j], px, py) == keep_min) { x[j] = px; y[j] = py; }
        }
        __syncthreads();
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const unsigned i = (unsigned)(G * j + t);
          const uint64_t px = __shfl_xor_sync(0xffffffffu, x[j], (int)st);
          const int32_t py = __shfl_xor_sync(0xffffffffu, y[j], (int)st);
          const bool keep_min = ((i & st) == 0) == ((i & s2) == 0);
          if (pair_gt(x[j], y[j], px, py) == keep_min) { x[j] = px; y[j] = py; }
        }
      }
    }
  }
}

// Sort the bucket [off, off + size) of (sk, si) with a group of G threads and emit its first
// `take` ids at out[off ...].
template <int E, int G>
__device__ __forceinline__ void sort_bucket(const SelArgs &a, const uint64_t *sk, const int32_t *si, unsigned off,
                                            unsigned size, unsigned take, uint64_t *sbk, int32_t *sbi) {
  const int t = G == 32 ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  uint64_t x[E];
  int32_t y[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(G * j + t);
    x[j] = i < size ? __ldcg(sk + off + i) : kInf;
    y[j] = i < size ? __ldcg(si + off + i) : INT32_MAX;
  }
  group_sort<E, G>(x, y, sbk, sbi);
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(G * j + t);
    if (i < take) emit(a, (int64_t)off + i, y[j]);
  }
}

// CTA bucket of <= E * kT pairs: one more MSD digit (the bucket's next digit ds) in shared
// memory, then each pair's rank inside its sub-bin by counting (the composite is unique, so the
// rank is the position): pairs land at off + sub-bin start + rank.  Sub-bins are ~1-3 pairs on
// spread keys; when one holds more than kSub the bucket is sorted by the bitonic network
// instead.  s_st = kBins + 1 counters (sub-bin slots, then their exclusive starts).
constexpr int kSub = 48;
template <int E>
__device__ __forceinline__ void radix_bucket(const SelArgs &a, const uint64_t *sk, const int32_t *si, unsigned off,
                                             unsigned size, unsigned take, const DigSel &ds, uint64_t *sbk,
                                             int32_t *sbi, unsigned *s_st, unsigned *s_w) {
  const int t = (int)threadIdx.x;
  uint64_t x[E];
  int32_t y[E];
  int d[E];
  unsigned slot[E];
#pragma unroll
  for (int u = 0; u < kPer; ++u) s_st[kPer * t + u] = 0u;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(kT * j + t);
    x[j] = i < size ? __ldcg(sk + off + i) : kInf;
    y[j] = i < size ? __ldcg(si + off + i) : INT32_MAX;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(kT * j + t);
    d[j] = i < size ? digit(ds, x[j], y[j]) : 0;
    slot[j] = i < size ? atomicAdd(&s_st[d[j]], 1u) : 0u;
  }
  __syncthreads();
  unsigned h[kPer], sum = 0;
  bool big = false;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    h[u] = s_st[kPer * t + u];
    sum += h[u];
    big |= h[u] > (unsigned)kSub;
  }
  unsigned tot;
  unsigned run = block_scan(sum, s_w, tot);  // ends with a barrier: every count read
  if (__syncthreads_or(big)) {
    group_sort<E, kT>(x, y, sbk, sbi);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const unsigned i = (unsigned)(kT * j + t);
      if (i < take) emit(a, (int64_t)off + i, y[j]);
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) { s_st[kPer * t + u] = run; run += h[u]; }
  if (t == 0) s_st[kBins] = size;
  __syncthreads();
  unsigned lo[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(kT * j + t);
    lo[j] = s_st[d[j]];
    if (i < size) { sbk[lo[j] + slot[j]] = x[j]; sbi[lo[j] + slot[j]] = y[j]; }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(kT * j + t);
    if (i >= size) continue;
    const unsigned hi = s_st[d[j] + 1];
    unsigned pos = lo[j];
    if (hi - lo[j] > 1u)
      for (unsigned q = lo[j]; q < hi; ++q) pos += pair_gt(x[j], y[j], sbk[q], sbi[q]) ? 1u : 0u;
    if (pos < take) emit(a, (int64_t)off + pos, y[j]);
  }
}

// Warp bucket of <= 32 * E pairs (E >= 2), the same scheme as radix_bucket with an 8-bit digit
// (the top bits of the bucket's next digit) in the warp's own shared-memory area; a sub-bin
// of more than kSubW pairs sends the bucket to the bitonic network.
constexpr int kWB = kT >= 512 ? 256 : 128;  // warp sub-bins (8- / 7-bit digit)
constexpr int kSubW = 24;
struct WarpArea {
  uint64_t k[kWarpMax];
  int32_t i[kWarpMax];
  unsigned h[kWB + 4];
};
// the round / CTA-bucket buffer: two bin arrays | a sort buffer + sub-bin starts
constexpr int kBufBase = (kCap * 12 > 8 * kBins ? kCap * 12 : 8 * kBins) + 4 * (kBins + 4);
// 256-thread builds keep the warp areas in that buffer (the small buckets run after the CTA
// ones): ~30 KB of shared memory per CTA in all, so the CTA shares its SM with two decode CTAs
constexpr bool kAliasWarp = kT <= 256;
constexpr int kWarpBytes = kNW * (int)sizeof(WarpArea);
constexpr int kBufBytes = kAliasWarp && kWarpBytes > kBufBase ? kWarpBytes : kBufBase;
constexpr int kDynBytes = kAliasWarp ? 0 : kWarpBytes;
template <int E>
__device__ __forceinline__ void warp_radix_bucket(const SelArgs &a, const uint64_t *sk, const int32_t *si,
                                                  unsigned off, unsigned size, unsigned take, DigSel ds,
                                                  WarpArea *wa) {
  constexpr int P = kWB / 32;
  const int lane = (int)(threadIdx.x & 31);
  constexpr int kWBits = kWB == 256 ? 8 : 7;  // the digit's top bits index the kWB sub-bins
  if (ds.w > kWBits) { ds.lo += ds.w - kWBits; ds.w = kWBits; }
  uint64_t x[E];
  int32_t y[E];
  int d[E];
  unsigned slot[E];
#pragma unroll
  for (int u = 0; u < P; ++u) wa->h[P * lane + u] = 0u;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(32 * j + lane);
    x[j] = i < size ? __ldcg(sk + off + i) : kInf;
    y[j] = i < size ? __ldcg(si + off + i) : INT32_MAX;
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(32 * j + lane);
    d[j] = i < size ? digit(ds, x[j], y[j]) : 0;
    slot[j] = i < size ? atomicAdd(&wa->h[d[j]], 1u) : 0u;
  }
  __syncwarp();
  unsigned h[P], sum = 0;
  bool big = false;
#pragma unroll
  for (int u = 0; u < P; ++u) {
    h[u] = wa->h[P * lane + u];
    sum += h[u];
    big |= h[u] > (unsigned)kSubW;
  }
  if (__any_sync(0xffffffffu, big)) {
    group_sort<E, 32>(x, y, nullptr, nullptr);
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const unsigned i = (unsigned)(32 * j + lane);
      if (i < take) emit(a, (int64_t)off + i, y[j]);
    }
    __syncwarp();
    return;
  }
  unsigned run = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, run, o);
    if (lane >= o) run += v;
  }
  run -= sum;
  __syncwarp();
#pragma unroll
  for (int u = 0; u < P; ++u) { wa->h[P * lane + u] = run; run += h[u]; }
  if (lane == 0) wa->h[kWB] = size;
  __syncwarp();
  unsigned lo[E];
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(32 * j + lane);
    lo[j] = wa->h[d[j]];
    if (i < size) { wa->k[lo[j] + slot[j]] = x[j]; wa->i[lo[j] + slot[j]] = y[j]; }
  }
  __syncwarp();
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const unsigned i = (unsigned)(32 * j + lane);
    if (i >= size) continue;
    const unsigned hi = wa->h[d[j] + 1];
    unsigned pos = lo[j];
    if (hi - lo[j] > 1u)
      for (unsigned q = lo[j]; q < hi; ++q) pos += pair_gt(x[j], y[j], wa->k[q], wa->i[q]) ? 1u : 0u;
    if (pos < take) emit(a, (int64_t)off + pos, y[j]);
  }
  __syncwarp();
}

#ifndef KVA_SEL_MAXREG
#define KVA_SEL_MAXREG 80  // measured: 1M keys alone 70 us (74 CTAs), co-runs with the attention
#endif
__global__ void __maxnreg__(KVA_SEL_MAXREG) evict_select_kernel(const __grid_constant__ SelArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ __align__(16) unsigned char s_buf[kBufBytes];
  extern __shared__ __align__(16) unsigned char s_dyn[];  // kNW WarpAreas (small buckets)
  __shared__ unsigned s_w[kNW];
  __shared__ unsigned long long s_red[3][kNW];
  __shared__ Comp s_comp;
  __shared__ unsigned s_bnd[4];
  unsigned *s_cnt = reinterpret_cast<unsigned *>(s_buf);  // [kBins] this CTA's counts per bin
  unsigned *s_off = s_cnt + kBins;                         // [kBins] its reserved offsets / cursors
  const int C = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  Ctl *ctl = a.ctl;
  int tp = 0;
  // diagnostics (-DKVA_SEL_SPAN): per-CTA end of the large buckets (part[c].o, thread 0) and
  // exit (part[c].pad, latest warp), %globaltimer ns
  auto span_mark = [&](bool at_exit) {
#ifdef KVA_SEL_SPAN
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!at_exit && tid == 0) a.part[c].o = t;
    if (at_exit && lane == 0) atomicMax(&a.part[c].pad, t);
#endif
  };
  auto stamp = [&]() {
    if (c == 0 && tid == 0 && tp < 32) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      ctl->t[tp] = t;
    }
    ++tp;
  };
  stamp();
  if (a.span && c == 0 && tid == 0) a.span[0] = gtime();
  auto span_end = [&]() {
    if (a.span) {
      __syncthreads();
      if (tid == 0) atomicMax(a.span + 1, gtime());
    }
  };
  const int64_t n = a.n;
  const int64_t per = (((n + C - 1) / C) + 3) & ~3ll;  // multiple of 4: 16-B aligned key / metadata slices
  const int64_t lo = std::min<int64_t>(n, c * per), hi = std::min<int64_t>(n, lo + per);
  const bool vec = (reinterpret_cast<uintptr_t>(a.keys) & 15) == 0;

  // Walk this CTA's slice of the input keys: f(key, id), 2 x 4 keys in flight per thread.
  // Walk this CTA's slice of the input keys, 4 keys per lane per call: f(key[4], id[4]) (kInf =
  // no key); a 4-deep register pipeline of 16-B loads (2 per call)
  auto for_slice = [&](auto &&f) {
    uint64_t k4[4];
    int32_t i4[4];
    if (vec) {
      const int64_t v0 = lo >> 1, v1 = hi >> 1;  // lo even
      const uint4 *src = reinterpret_cast<const uint4 *>(a.keys);
      auto ld = [&](int64_t i) { return i < v1 ? __ldcg(src + i) : make_uint4(~0u, ~0u, ~0u, ~0u); };
      uint4 q0 = ld(v0 + tid), q1 = ld(v0 + kT + tid), q2 = ld(v0 + 2 * kT + tid), q3 = ld(v0 + 3 * kT + tid);
#pragma unroll 1
      for (int64_t b = v0; b < v1; b += 2 * kT) {
        const uint4 x = q0, y = q1;
        q0 = q2;
        q1 = q3;
        q2 = ld(b + 4 * kT + tid);
        q3 = ld(b + 5 * kT + tid);
        const int64_t i = b + tid, j = b + kT + tid;
        k4[0] = ((uint64_t)x.y << 32) | x.x;
        k4[1] = ((uint64_t)x.w << 32) | x.z;
        k4[2] = ((uint64_t)y.y << 32) | y.x;
        k4[3] = ((uint64_t)y.w << 32) | y.z;
        i4[0] = (int32_t)(2 * i);
        i4[1] = (int32_t)(2 * i + 1);
        i4[2] = (int32_t)(2 * j);
        i4[3] = (int32_t)(2 * j + 1);
        f(k4, i4);
      }
      if ((hi & 1) && hi > lo) {  // odd tail of the last slice: thread 0 of a full warp pass
        k4[0] = tid == 0 ? a.keys[hi - 1] : kInf;
        k4[1] = k4[2] = k4[3] = kInf;
        i4[0] = i4[1] = i4[2] = i4[3] = (int32_t)(hi - 1);
        f(k4, i4);
      }
    } else {
      for (int64_t b = lo; b < hi; b += 4 * kT) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t i = b + u * kT + tid;
          k4[u] = i < hi ? a.keys[i] : kInf;
          i4[u] = (int32_t)i;
        }
        f(k4, i4);
      }
    }
  };

  if (a.fused) {  // the KV-manager step's phases 0-2 (internal.h), then its keys pass in phase 0
    manager_phases(a.mgr, (int64_t)c * kT + tid, (int64_t)C * kT, [&] { stamp(); grid.sync(); stamp(); },
                   reinterpret_cast<int32_t *>(s_buf), kBufBytes / 4);
    stamp();
  }
  // ---------------- phase 0: which bits vary among the evictable keys, how many ----------------
  // The pass also counts digit 0 speculatively, with the layout of the varying-bit mask the
  // previous call on this workspace found (ctl->v_prev; any value is safe: the counts are used
  // only when it equals this call's mask, else phase 1 counts again).
  {
    if (tid == 0) make_comp(s_comp, __ldcg(&ctl->v_prev), n);
    for (int i = tid; i < kBins; i += kT) s_cnt[i] = 0u;
    __syncthreads();
    const Comp &cg0 = s_comp;
    const Dig0R d0r = dig0_regs(cg0);
    const CompR cr0 = comp_regs(cg0);
    const DigSel ds0 = dig_sel(cg0, 0);
    const bool raw0 = d0r.n0 >= 0;
    unsigned long long o = 0, an = 0, cn = 0;
    stamp();
    auto acc = [&](const uint64_t (&k4)[4], const int32_t (&i4)[4]) {
      int d4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k4[u] != kInf) {
          o |= k4[u];
          an |= ~k4[u];
          ++cn;
        }
        d4[u] = k4[u] == kInf ? -1 : raw0 ? digit0_raw(d0r, k4[u]) : digit(ds0, compress(cr0, k4[u]), i4[u]);
      }
      hist_batch<4>(s_cnt, d4);
    };
    if (a.fused) {  // the manager's keys pass over this CTA's slice, feeding the statistics
      const MgrArgs &m = a.mgr;
      uint64_t *keys_out = m.keys;
      unsigned act = 0;
      const bool mvec = (lo & 3) == 0 &&
                        ((reinterpret_cast<uintptr_t>(m.state) | reinterpret_cast<uintptr_t>(m.rc) |
                          reinterpret_cast<uintptr_t>(m.lat) | reinterpret_cast<uintptr_t>(keys_out) |
                          (m.depth ? reinterpret_cast<uintptr_t>(m.depth) : 0)) & 15) == 0;
      const int64_t q0 = lo >> 2, q1 = mvec ? (hi >> 2) : q0;
      for (int64_t base = q0; base < q1; base += kT) {  // 4 blocks per lane, vector loads / stores
        const int64_t q = base + tid;
        uint64_t k4[4] = {kInf, kInf, kInf, kInf};
        int32_t i4[4];
        if (q < q1) {
          const uint32_t s4 = __ldcg(reinterpret_cast<const uint32_t *>(m.state) + q);
          const uint4 r4 = __ldcg(reinterpret_cast<const uint4 *>(m.rc) + q);
          const uint4 l4 = __ldcg(reinterpret_cast<const uint4 *>(m.lat) + q);
          uint2 dd = make_uint2(0u, 0u);
          if (m.depth) dd = __ldcg(reinterpret_cast<const uint2 *>(m.depth) + q);
          k4[0] = manager_key(s4 & 0xFF, r4.x, l4.x, dd.x & 0xFFFF, act);
          k4[1] = manager_key((s4 >> 8) & 0xFF, r4.y, l4.y, dd.x >> 16, act);
          k4[2] = manager_key((s4 >> 16) & 0xFF, r4.z, l4.z, dd.y & 0xFFFF, act);
          k4[3] = manager_key(s4 >> 24, r4.w, l4.w, dd.y >> 16, act);
          reinterpret_cast<ulonglong2 *>(keys_out)[2 * q] = make_ulonglong2(k4[0], k4[1]);
          reinterpret_cast<ulonglong2 *>(keys_out)[2 * q + 1] = make_ulonglong2(k4[2], k4[3]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) i4[u] = (int32_t)(4 * q + u);
        acc(k4, i4);
      }
      for (int64_t b0 = std::max<int64_t>(lo, 4 * q1); b0 < hi; b0 += kT) {  // scalar rest of the slice
        const int64_t i = b0 + tid;
        uint64_t k4[4] = {kInf, kInf, kInf, kInf};
        const int32_t i4[4] = {(int32_t)i, (int32_t)i, (int32_t)i, (int32_t)i};
        if (i < hi) {
          k4[0] = manager_key(__ldcg(m.state + i), __ldcg(m.rc + i), __ldcg(m.lat + i), m.depth ? m.depth[i] : 0u, act);
          keys_out[i] = k4[0];
        }
        acc(k4, i4);
      }
      if (m.n_active) {  // one atomic per warp
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) act += __shfl_xor_sync(0xffffffffu, act, s);
        if (lane == 0 && act) atomicAdd(m.n_active, (unsigned long long)act);
      }
    } else {
      for_slice(acc);
    }
    stamp();
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      o |= __shfl_xor_sync(0xffffffffu, o, s);
      an |= __shfl_xor_sync(0xffffffffu, an, s);
      cn += __shfl_xor_sync(0xffffffffu, cn, s);
    }
    if (lane == 0) { s_red[0][w] = o; s_red[1][w] = an; s_red[2][w] = cn; }
    __syncthreads();
    if (tid == 0) {
      Part p{0, 0, 0, 0};
      for (int i = 0; i < kNW; ++i) { p.o |= s_red[0][i]; p.a |= s_red[1][i]; p.c += s_red[2][i]; }
      a.part[c] = p;
    }
    for (int i = c * kT + tid; i < 2 * kBins; i += C * kT) a.hist[i] = 0u;  // digit-0 and -1 counts
    if (c == 0 && tid < kMaxLevels) {
      ctl->n_small[tid] = 0u;
      ctl->n_large[tid] = 0u;
      ctl->n_big[tid] = 0u;
    }
  }
  stamp();
  grid.sync();
  stamp();

  // ---------------- phase 1: composite layout + digit-0 histogram ----------------
  unsigned long long E;
  bool hit;
  {
    unsigned long long o = 0, an = 0, cn = 0;
    if (tid < C) {
      const Part p = a.part[tid];
      o = p.o; an = p.a; cn = p.c;
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      o |= __shfl_xor_sync(0xffffffffu, o, s);
      an |= __shfl_xor_sync(0xffffffffu, an, s);
      cn += __shfl_xor_sync(0xffffffffu, cn, s);
    }
    if (lane == 0) { s_red[0][w] = o; s_red[1][w] = an; s_red[2][w] = cn; }
    __syncthreads();
    if (tid == 0) {
      unsigned long long O = 0, A = 0, N = 0;
      for (int i = 0; i < kNW; ++i) { O |= s_red[0][i]; A |= s_red[1][i]; N += s_red[2][i]; }
      const uint64_t V = O & A;  // set in some evictable key and clear in another
      const bool h = V == s_comp.v;
      if (!h) make_comp(s_comp, V, n);
      unsigned long long mall = 0;
      for (int i = 0; i < s_comp.nr; ++i) mall |= s_comp.mask[i];
      s_comp.cst = O & ~A & ~mall;
      s_red[2][0] = N;
      s_red[1][0] = h ? 1ull : 0ull;
      if (c == 0) {
        *a.d_count = (int64_t)std::min<unsigned long long>(N, (unsigned long long)a.k);
        ctl->v_prev = V;  // every CTA read the old value before the barrier
      }
    }
    __syncthreads();
    E = s_red[2][0];
    hit = s_red[1][0] != 0ull;
  }
  if (E == 0) {  // uniform: nothing evictable (*d_count = 0)
    span_end();
    return;
  }
  const Comp &cp = s_comp;
  const CompR cr = comp_regs(cp);
  if (!hit) {  // the layout changed: count digit 0 again
    for (int i = tid; i < kBins; i += kT) s_cnt[i] = 0u;
    const DigSel ds0 = dig_sel(cp, 0);
    __syncthreads();
    const Dig0R d0r = dig0_regs(cp);
    const bool raw0 = d0r.n0 >= 0;
    for_slice([&](const uint64_t (&k4)[4], const int32_t (&i4)[4]) {
      int d4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        d4[u] = k4[u] == kInf ? -1 : raw0 ? digit0_raw(d0r, k4[u]) : digit(ds0, compress(cr, k4[u]), i4[u]);
      hist_batch<4>(s_cnt, d4);
    });
    __syncthreads();
  }
  stamp();
  flush_counts(s_cnt, s_off, a.hist);
  stamp();
  grid.sync();
  stamp();

  // ---------------- rounds: partition the segment holding rank k-1 ----------------
  const unsigned long long kk = (unsigned long long)a.k;
  bool full = E <= kk;                 // the whole segment is taken
  unsigned long long need = full ? E : kk;
  unsigned out_base = 0;
  unsigned m_lo = 0, m_cnt = 0;        // rounds >= 1: this CTA's range of the segment in wk/wi
  unsigned rec_small = 0, rec_large = 0;  // CTA 0: level-0 records appended so far
  int r = 0;
  for (;; ++r) {
    const unsigned *Hr = a.hist + (r % 3) * kBins;
    {  // zero the digit-(r+2) counts (last read in round r-1)
      unsigned *Hz = a.hist + ((r + 2) % 3) * kBins;
      for (int i = c * kT + tid; i < kBins; i += C * kT) Hz[i] = 0u;
    }
    unsigned h[kPer], ex[kPer];
    unsigned sum = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      h[u] = __ldcg(Hr + kPer * tid + u);
      sum += h[u];
    }
    unsigned tot;
    unsigned run = block_scan(sum, s_w, tot);
#pragma unroll
    for (int u = 0; u < kPer; ++u) { ex[u] = run; run += h[u]; }
    if (!full) {
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if ((unsigned long long)ex[u] < need && need <= (unsigned long long)ex[u] + h[u]) {
          s_bnd[0] = kPer * tid + u;
          s_bnd[1] = ex[u];
          s_bnd[2] = h[u];
        }
    }
    __syncthreads();
    // bin categories: [0, sure_end) taken; bin b: finish-sort (fin) or next segment (nxt)
    int b = kBins, sure_end = kBins;
    bool fin = false, nxt = false;
    unsigned long long need_b = 0;
    unsigned less_b = 0, h_b = 0;
    if (!full) {
      b = (int)s_bnd[0];
      less_b = s_bnd[1];
      h_b = s_bnd[2];
      need_b = need - less_b;
      if (need_b == h_b) sure_end = b + 1;
      else {
        sure_end = b;
        if (h_b <= (unsigned)kCap) fin = true;
        else nxt = true;
      }
    }
    const unsigned m_lo_next = nxt ? s_off[b] : 0u, m_cnt_next = nxt ? s_cnt[b] : 0u;
    __syncthreads();
    // absolute destinations: taken / finished bins -> output-aligned staging (bit 31: a
    // singleton bin, emitted directly); the next segment -> wk/wi from 0
    unsigned nrec = 0;  // this thread's level-0 bucket records: small count | large count << 16
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int d = kPer * tid + u;
      const bool tk = d < sure_end || (fin && d == b);
      if (tk) s_off[d] += (out_base + ex[u]) | (h[u] == 1u && d < sure_end ? 0x80000000u : 0u);
      if (tk && h[u] >= 2u) nrec += h[u] <= (unsigned)kWarpMax ? 1u : 0x10000u;
    }
    if (c == 0) {  // CTA 0 alone appends the rounds' records: running totals, no atomics
      unsigned tot_rec;
      unsigned at = block_scan(nrec, s_w, tot_rec);
      unsigned at_s = rec_small + (at & 0xFFFFu), at_l = rec_large + (at >> 16);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int d = kPer * tid + u;
        if ((d < sure_end || (fin && d == b)) && h[u] >= 2u) {
          const unsigned take = d < sure_end ? h[u] : (unsigned)need_b;
          const uint4 rec = make_uint4(out_base + ex[u], h[u], take, (unsigned)(r + 1));
          if (h[u] <= (unsigned)kWarpMax) a.rs[0][at_s++] = rec;
          else {
            a.rl[0][at_l++] = rec;
            if (h[u] > (unsigned)kCap) atomicAdd(&ctl->n_big[0], 1u);
          }
        }
      }
      rec_small += tot_rec & 0xFFFFu;
      rec_large += tot_rec >> 16;
      if (tid == 0) {
        ctl->n_small[0] = rec_small;
        ctl->n_large[0] = rec_large;
      }
    }
    if (nxt)
      for (int i = tid; i < kBins; i += kT) s_cnt[i] = 0u;  // digit-(r+1) counts of the next segment
    if (tid == 0) s_bnd[3] = 0u;  // round 0: this CTA's compacted pair count
    __syncthreads();

    stamp();
    const int wsrc = r & 1, wdst = (r + 1) & 1;
    const DigSel dsr = dig_sel(cp, r), dsn = dig_sel(cp, r + 1);
    // NK (compressed key, id) pairs per lane: digit, category, batched position claim, store,
    // and the next segment's digit-(r+1) count
    auto place = [&](auto nkc, const uint64_t *key, const int32_t *id, const bool *valid) {
      constexpr int NK = decltype(nkc)::value;
      int d[NK], dn[NK];
      unsigned pos[NK];
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        d[k] = valid[k] ? digit(dsr, key[k], id[k]) : -1;
        const bool taken = d[k] >= 0 && (d[k] < sure_end || (fin && d[k] == b));
        const bool seg = nxt && d[k] == b;
        if (!taken && !seg) d[k] = -1;
        dn[k] = seg && d[k] >= 0 ? digit(dsn, key[k], id[k]) : -1;
      }
      claim_batch<NK>(s_off, d, pos);
#pragma unroll
      for (int k = 0; k < NK; ++k) {
        if (d[k] < 0) continue;
        if (nxt && d[k] == b) {
          a.wk[wdst][pos[k]] = key[k];
          a.wi[wdst][pos[k]] = id[k];
        } else if (pos[k] & 0x80000000u) {
          emit(a, pos[k] & 0x7FFFFFFFu, id[k]);
        } else {
          a.sk[0][pos[k]] = key[k];
          a.si[0][pos[k]] = id[k];
        }
      }
      hist_batch<NK>(s_cnt, dn);
    };
    // place a segment [xk, xk + cnt) of (compressed key, id) pairs, 2 per lane per pass
    // (raw: the pairs hold input keys, compressed here)
    auto seg_loop = [&](const uint64_t *xk, const int32_t *xi, unsigned cnt, bool raw) {
      for (unsigned base = 0; base < cnt; base += 2 * kT) {
        const unsigned i0 = base + tid, i1 = base + kT + tid;
        const bool v0 = i0 < cnt, v1 = i1 < cnt;
        uint64_t k2[2] = {v0 ? __ldcg(xk + i0) : kInf, v1 ? __ldcg(xk + i1) : kInf};
        if (raw) {
          k2[0] = v0 ? compress(cr, k2[0]) : kInf;
          k2[1] = v1 ? compress(cr, k2[1]) : kInf;
        }
        const int32_t d2[2] = {v0 ? __ldcg(xi + i0) : 0, v1 ? __ldcg(xi + i1) : 0};
        const bool b2[2] = {v0, v1};
        place(std::integral_constant<int, 2>{}, k2, d2, b2);
      }
    };
    if (r == 0) {
      // keys above bin b are dropped before compressing: digit > b <=> key >= t_hi (compress is
      // an order isomorphism on keys that agree outside the runs; t_hi = the smallest such key
      // whose compressed value has digit b + 1), when digit 0 lies within the key bits
      uint64_t t_hi = kInf;
      if (!full && dsr.lo >= cp.idb) {
        const int sh = dsr.lo - cp.idb, kb = cp.B - cp.idb;  // compressed key bits
        const uint64_t x = (uint64_t)(b + 1) << sh;
        if (sh + dsr.w < kb || (kb < 64 && x < (1ull << kb))) {
          uint64_t t = cp.cst;
          for (int i = 0; i < cp.nr; ++i) t |= (x << cp.sh[i]) & cp.mask[i];
          t_hi = t;
        }
      }
      // filter, then place: the keys below t_hi (typically a small fraction) are compacted
      // (raw; compressed when placed) into this CTA's own range of wk[0] (one shared atomic per warp pass, ballot
      // ranks); the dropped keys cost a compare and a ballot.  The CTA then places its compacted
      // pairs like a later round's segment: every lane busy, no grid barrier in between (the
      // pairs stay with the CTA that counted them, so its bin reservations still hold).
      uint64_t *ck = a.wk[0] + lo;
      int32_t *ci = a.wi[0] + lo;
      const unsigned lt = lanemask_lt();
      for_slice([&](const uint64_t (&k4)[4], const int32_t (&i4)[4]) {
        bool v[4];
        unsigned m[4], tot = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          v[u] = k4[u] < t_hi;  // also excludes kInf
          m[u] = __ballot_sync(0xffffffffu, v[u]);
          tot += __popc(m[u]);
        }
        if (tot == 0u) return;
        unsigned at = 0;
        if (lane == 0) at = atomicAdd(&s_bnd[3], tot);
        at = __shfl_sync(0xffffffffu, at, 0);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (v[u]) {
            const unsigned p = at + __popc(m[u] & lt);
            ck[p] = k4[u];
            ci[p] = i4[u];
          }
          at += __popc(m[u]);
        }
      });
      stamp();
      __syncthreads();
      seg_loop(ck, ci, s_bnd[3], true);
    } else {
      stamp();  // (keeps the stamp count per round equal)
      seg_loop(a.wk[wsrc] + m_lo, a.wi[wsrc] + m_lo, m_cnt, false);
    }
    stamp();
    if (nxt) {  // reserve this CTA's ranges in the next segment's digit bins
      __syncthreads();
      unsigned *Hn = a.hist + ((r + 1) % 3) * kBins;
      flush_counts(s_cnt, s_off, Hn);
      need = need_b;
      out_base += less_b;
      m_lo = m_lo_next;
      m_cnt = m_cnt_next;
    }
    stamp();
    grid.sync();
    stamp();
    if (!nxt) break;
  }
  if (c == 0 && tid == 0) ctl->rounds = (unsigned)(r + 1);

  // ---------------- buckets: sort every taken bin of >= 2 pairs ----------------
  uint64_t *sbk = reinterpret_cast<uint64_t *>(s_buf);
  int32_t *sbi = reinterpret_cast<int32_t *>(s_buf + kCap * 8);
  unsigned *s_st = reinterpret_cast<unsigned *>(s_buf + (kCap * 12 > 8 * kBins ? kCap * 12 : 8 * kBins));
  for (int lv = 0; lv < kMaxLevels; ++lv) {
    const int L = lv & 1;
    const unsigned nl = __ldcg(&ctl->n_large[lv]), ns = __ldcg(&ctl->n_small[lv]);
    const bool more = __ldcg(&ctl->n_big[lv]) != 0u;
    for (unsigned ri = c; ri < nl; ri += C) {
      const uint4 rec = __ldcg(a.rl[L] + ri);
      const unsigned off = rec.x, size = rec.y, take = rec.z, dg = rec.w & 0xFF, src = rec.w >> 8;
      const uint64_t *xk = a.sk[src];
      const int32_t *xi = a.si[src];
      if (size <= (unsigned)kCap) {  // the CTA: one more digit in shared memory + sub-bin ranks
        const DigSel dsb = dig_sel(cp, dg);
        if (size <= (unsigned)kT) {
          radix_bucket<1>(a, xk, xi, off, size, take, dsb, sbk, sbi, s_st, s_w);
        } else if (size <= 2u * kT) {
          radix_bucket<2>(a, xk, xi, off, size, take, dsb, sbk, sbi, s_st, s_w);
        } else {
          if constexpr (kCap > 2 * kT) radix_bucket<kCap / kT>(a, xk, xi, off, size, take, dsb, sbk, sbi, s_st, s_w);
        }
        __syncthreads();
      } else {  // partition by the next digit into the other staging buffer -> next level
        uint64_t *yk = a.sk[src ^ 1];
        int32_t *yi = a.si[src ^ 1];
        const DigSel dsp = dig_sel(cp, dg);
        for (int i = tid; i < kBins; i += kT) s_cnt[i] = 0u;
        __syncthreads();
        for (unsigned base = 0; base < size; base += kT) {
          const unsigned i = base + tid;
          hist_add(s_cnt, i < size ? digit(dsp, __ldcg(xk + off + i), __ldcg(xi + off + i)) : -1);
        }
        __syncthreads();
        unsigned hh[kPer], sm = 0;
#pragma unroll
        for (int u = 0; u < kPer; ++u) { hh[u] = s_cnt[kPer * tid + u]; sm += hh[u]; }
        unsigned tt;
        unsigned rr = block_scan(sm, s_w, tt);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int d = kPer * tid + u;
          s_off[d] = (off + rr) | (hh[u] == 1u ? 0x80000000u : 0u);
          if (hh[u] >= 2u) {
            const uint4 r2 = make_uint4(off + rr, hh[u], hh[u], (unsigned)(dg + 1) | ((src ^ 1u) << 8));
            if (hh[u] <= (unsigned)kWarpMax) {
              a.rs[L ^ 1][atomicAdd(&ctl->n_small[lv + 1], 1u)] = r2;
            } else {
              a.rl[L ^ 1][atomicAdd(&ctl->n_large[lv + 1], 1u)] = r2;
              if (hh[u] > (unsigned)kCap) atomicAdd(&ctl->n_big[lv + 1], 1u);
            }
          }
          rr += hh[u];
        }
        __syncthreads();
        for (unsigned base = 0; base < size; base += kT) {
          const unsigned i = base + tid;
          const bool v = i < size;
          const uint64_t key = v ? __ldcg(xk + off + i) : 0ull;
          const int32_t id = v ? __ldcg(xi + off + i) : 0;
          const unsigned pos = bin_claim(s_off, v ? digit(dsp, key, id) : -1);
          if (v) {
            if (pos & 0x80000000u) emit(a, pos & 0x7FFFFFFFu, id);
            else { yk[pos] = key; yi[pos] = id; }
          }
        }
        __syncthreads();
      }
    }
    stamp();
    if (!more) span_mark(false);
    // small buckets on the CTAs without a large one (all CTAs when every CTA had one), spread
    // over CTAs first: with fewer large buckets than CTAs the two kinds run side by side
    {
      const unsigned nl0 = nl < (unsigned)C ? nl : 0u, Cs = (unsigned)C - nl0;
      WarpArea *wa = reinterpret_cast<WarpArea *>(kAliasWarp ? s_buf : s_dyn) + w;
      if ((unsigned)c >= nl0)
        for (unsigned ri = (unsigned)w * Cs + ((unsigned)c - nl0); ri < ns; ri += (unsigned)kNW * Cs) {
          const uint4 rec = __ldcg(a.rs[L] + ri);
          const unsigned off = rec.x, size = rec.y, take = rec.z, dg = rec.w & 0xFF, src = rec.w >> 8;
          const DigSel dsb = dig_sel(cp, dg);
          if (size <= 32) sort_bucket<1, 32>(a, a.sk[src], a.si[src], off, size, take, nullptr, nullptr);
          else if (size <= 64) warp_radix_bucket<2>(a, a.sk[src], a.si[src], off, size, take, dsb, wa);
          else if (size <= 128) warp_radix_bucket<4>(a, a.sk[src], a.si[src], off, size, take, dsb, wa);
          else warp_radix_bucket<8>(a, a.sk[src], a.si[src], off, size, take, dsb, wa);
        }
    }
    stamp();
    if (!more) {
      if (c == 0 && tid == 0) ctl->levels = (unsigned)(lv + 1);
      span_mark(true);
      span_end();
      break;
    }
    grid.sync();
    stamp();
  }
}

}  // namespace

size_t KVA_SEL_CAT(evict_select_ws_bytes_, KVA_SEL_VARIANT)(int64_t n, int64_t k) { return layout(n, k).total; }

cudaError_t KVA_SEL_CAT(launch_evict_select_, KVA_SEL_VARIANT)(const uint64_t *keys, int64_t n, int64_t k,
                                                               int32_t *out_ids, int64_t *d_count, uint32_t *free_bits,
                                                               void *ws, size_t ws_bytes, int ctas, cudaStream_t s,
                                                               const MgrArgs *mgr) {
  const Layout L = layout(n, k);
  if (ws_bytes < L.total) return cudaErrorInvalidValue;
  uint8_t *p = static_cast<uint8_t *>(ws);
  SelArgs a{};
  a.keys = keys;
  a.n = n;
  a.k = k;
  a.out_ids = out_ids;
  a.d_count = d_count;
  a.free_bits = free_bits;
  a.span = span_ring_slot(1);
  a.fused = mgr != nullptr;
  if (mgr) a.mgr = *mgr;
  a.ctl = reinterpret_cast<Ctl *>(p + L.ctl);
  a.part = reinterpret_cast<Part *>(p + L.part);
  a.hist = reinterpret_cast<unsigned int *>(p + L.hist);
  for (int i = 0; i < 2; ++i) {
    a.wk[i] = reinterpret_cast<uint64_t *>(p + L.wk[i]);
    a.wi[i] = reinterpret_cast<int32_t *>(p + L.wi[i]);
    a.sk[i] = reinterpret_cast<uint64_t *>(p + L.sk[i]);
    a.si[i] = reinterpret_cast<int32_t *>(p + L.si[i]);
    a.rs[i] = reinterpret_cast<uint4 *>(p + L.rs[i]);
    a.rl[i] = reinterpret_cast<uint4 *>(p + L.rl[i]);
  }
  const int nsm = sm_count();
  cudaError_t e = smem_attrs_once(reinterpret_cast<const void *>(evict_select_kernel), kDynBytes);
  if (e != cudaSuccess) return e;
  static const int per_sm = [] {  // co-resident CTAs per SM (cooperative launch bound)
    int v = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, evict_select_kernel, kT, kDynBytes);
    return std::max(1, v);
  }();
  int C = ctas > 0 ? ctas : nsm / 2;
  C = std::max(1, std::min(C, std::min(kMaxC, per_sm * nsm)));
  void *args[] = {(void *)&a};
  return cudaLaunchCooperativeKernel((void *)evict_select_kernel, dim3(C), dim3(kT), args, kDynBytes, s);
}

}  // namespace kva
