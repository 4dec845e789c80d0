// kernels_evict.cu — task-aware eviction: priority keys and the radix
// top-k that replaces the paper's host-side free-table priority queue.
//
// Order: "When evicting the KV cache, we will first consider the priority of the KV cache
// entry, and then the last access time"; priorities P:331-334.  Keys are
// order-preserving u64 codes (readings #18-#20); equal keys are broken by block id.
//
// evict_select is one cooperative persistent kernel (grid = #SMs, 1024 threads, keys of a
// CTA's slice cached in shared memory):
//   1. MSD radix select, 8 rounds of 8-bit digits -> the k-th smallest evictable key T and
//      count(< T);
//   2. order-preserving compaction of {key < T} u {first k - count(<T) blocks with key == T}
//      (block-id order) into a (key, id) array;
//   3. stable LSD radix sort of that array by key over only the bytes that vary (stability
//      keeps block-id order among equal keys).
// Grid-wide steps are separated by cooperative-groups grid barriers.
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace cg = cooperative_groups;

namespace kva {

constexpr uint64_t kInf = ~0ull;

__global__ void evict_keys_kernel(const uint8_t *__restrict__ state, const uint32_t *__restrict__ rc,
                                  const uint32_t *__restrict__ lat, const uint16_t *__restrict__ depth,
                                  int64_t n, uint64_t *__restrict__ keys) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s = state[b];
    uint64_t key;
    if (s == 0 || s == 1 || s == 2 || s > 5) {
      key = kInf;  // free / running online (priority inf) / pinned / unknown
    } else {
      const uint32_t r = rc[b];
      uint64_t code;
      if (r > 0) code = r >= 0x7FFFu ? 0xFFFEull : 2ull * r;  // priority rc
      else code = (s == 4) ? 1ull : 0ull;                      // 0.5 / 0
      const uint64_t dep = depth ? (uint64_t)depth[b] : 0ull;
      key = (code << 48) | ((uint64_t)lat[b] << 16) | (0xFFFFull - dep);
    }
    keys[b] = key;
  }
}

cudaError_t launch_evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                              const uint16_t *depth, int64_t n, uint64_t *keys, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 8);
  evict_keys_kernel<<<grid, 256, 0, s>>>(state, rc, lat, depth, n, keys);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
namespace {
constexpr int kThreads = 512;  // leaves registers/smem for a co-resident decode CTA
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCtas = 1024;
constexpr int kCandCap = 65535;  // candidate lists use u16 slice indices

struct SelWs {  // global scratch (zeroed by the host before launch)
  unsigned long long t[32];      // phase timestamps of CTA 0 (%globaltimer, ns; diagnostics)
  unsigned long long hist[8][256];
  unsigned long long cnt_eq[kMaxCtas], cnt_sel[kMaxCtas];
  unsigned long long key_or, key_and_inv;  // OR of selected keys, OR of their complements
};
struct SortWs {
  unsigned int hist[kMaxCtas][256];  // per-CTA digit counts of one LSD pass
};
}  // namespace

size_t evict_select_ws_bytes(int64_t n, int64_t k) {
  (void)n;
  const size_t pairs = (size_t)std::max<int64_t>(k, 1);
  return sizeof(SelWs) + sizeof(SortWs) + 2 * pairs * (sizeof(uint64_t) + sizeof(int32_t)) + 256;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one value per thread; `total` gets the block sum.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *s_warp, T &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    T t = lane < kWarps ? s_warp[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;  // inclusive prefix over warps
  }
  __syncthreads();
  total = s_warp[kWarps - 1];
  const T res = x - v + (w > 0 ? s_warp[w - 1] : T(0));
  __syncthreads();
  return res;
}

// Histogram increment with a fast path for warps whose 32 digits are equal (the common case
// for skewed keys): one atomic of 32 instead of 32 serialised same-address atomics.
__device__ __forceinline__ void hist_add_fast(unsigned int *hist, int dg) {
  const int d0 = __shfl_sync(0xffffffffu, dg, 0);
  if (__all_sync(0xffffffffu, dg == d0)) {
    if ((threadIdx.x & 31) == 0 && d0 < 256) atomicAdd(&hist[d0], 32u);
  } else if (dg < 256) {
    atomicAdd(&hist[dg], 1u);
  }
}

// Warp-aggregated shared-memory histogram increment (digit 256 = skip): one atomic per
// distinct digit per warp instead of one per lane (keys are highly skewed: e.g. the priority
// code byte is identical for most blocks).
__device__ __forceinline__ void warp_hist_add(unsigned int *hist, int dg) {
  const unsigned peers = __match_any_sync(0xffffffffu, dg);
  if (dg < 256 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
}

// Sum over threads of a u64 (result valid in all threads).
__device__ __forceinline__ unsigned long long block_sum(unsigned long long a,
                                                        unsigned long long *s_red) {
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = a;
  __syncthreads();
  unsigned long long t = 0;
  for (int w = 0; w < kWarps; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kThreads, 2)
    evict_select_kernel(const uint64_t *__restrict__ keys, int64_t n, int64_t k,
                        int32_t *__restrict__ out_ids, int64_t *__restrict__ d_count,
                        SelWs *__restrict__ sw, SortWs *__restrict__ so, uint64_t *pk0,
                        int32_t *pi0, uint64_t *pk1, int32_t *pi1, int cache_keys) {
  cg::grid_group grid = cg::this_grid();
  int tp = 0;
  auto stamp = [&]() {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (tp < 32) sw->t[tp] = t;
    }
    ++tp;
  };
  stamp();
  extern __shared__ uint64_t s_keys[];
  __shared__ unsigned int s_hist[256];
  __shared__ unsigned int s_base[256];
  __shared__ int s_warp[32];
  __shared__ long long s_warp64[32];
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_sel[4];
  __shared__ __align__(16) unsigned int s_wcnt[kWarps][256];  // 16 KB
  const int C = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int64_t per = (n + C - 1) / C;
  const int64_t lo = std::min<int64_t>(n, c * per), hi = std::min<int64_t>(n, lo + per);
  const int64_t cnt = hi - lo;
  // candidate index lists (u16, double-buffered) after the cached keys: every select round
  // scans only the keys still matching the chosen digit prefix
  const bool use_cand = cache_keys && per <= kCandCap;
  uint16_t *cand[2] = {reinterpret_cast<uint16_t *>(s_keys + (cache_keys ? per : 0)), nullptr};
  cand[1] = cand[0] + per;
  __shared__ int s_ncand[2];
  if (tid == 0) s_ncand[0] = s_ncand[1] = 0;
  __syncthreads();
  for (int64_t base = 0; base < cnt; base += kThreads) {
    const int64_t i = base + tid;
    uint64_t x = kInf;
    if (i < cnt) {
      x = keys[lo + i];
      if (cache_keys) s_keys[i] = x;
    }
    if (use_cand) {  // initial candidates: every evictable key (warp-aggregated append)
      const bool keep = x != kInf;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      int off = 0;
      if ((tid & 31) == 0 && bal) off = atomicAdd(&s_ncand[0], __popc(bal));
      off = __shfl_sync(0xffffffffu, off, 0);
      if (keep) cand[0][off + __popc(bal & lanemask_lt())] = (uint16_t)i;
    }
  }
  __syncthreads();
  auto key_at = [&](int64_t i) -> uint64_t { return cache_keys ? s_keys[i] : keys[lo + i]; };
  stamp();  // 1: keys cached

  // ---------------- 1. radix select: T = k-th smallest evictable key ----------------
  // 8 rounds of 8-bit digits: warp-aggregated shared-memory histograms (keys are heavily
  // skewed, e.g. the priority byte), one global atomic per (CTA, bin), grid barrier, then
  // every CTA scans the 256 global bins block-wide and the owner of rank kr publishes.
  uint64_t prefix = 0;
  unsigned long long kr = (unsigned long long)k, less = 0, total_ev = 0;
  bool take_all = false;
  int cb = 0;  // current candidate buffer
  for (int r = 0; r < 8; ++r) {
    const int shift = 56 - 8 * r;
    for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    const int64_t scan_n = use_cand ? s_ncand[cb] : cnt;
    for (int64_t base = 0; base < scan_n; base += kThreads) {  // warp-uniform trip count
      const int64_t i = base + tid;
      int dg = 256;  // sentinel: not a candidate
      if (i < scan_n) {
        const uint64_t x = key_at(use_cand ? (int64_t)cand[cb][i] : i);
        if (x != kInf && (r == 0 || (x >> (shift + 8)) == prefix)) dg = (int)((x >> shift) & 0xFF);
      }
      hist_add_fast(s_hist, dg);
    }
    __syncthreads();
    for (int i = tid; i < 256; i += kThreads)
      if (s_hist[i]) atomicAdd(&sw->hist[r][i], (unsigned long long)s_hist[i]);
    stamp();
    grid.sync();
    stamp();
    {
      const int h = tid < 256 ? (int)sw->hist[r][tid] : 0;
      int tot;
      const int excl = block_excl_scan(h, s_warp, tot);
      if (r == 0) {
        total_ev = (unsigned long long)tot;
        take_all = total_ev <= kr;
      }
      if (!take_all && tid < 256 && (unsigned long long)excl < kr && kr <= (unsigned long long)(excl + h)) {
        s_sel[0] = (prefix << 8) | (uint64_t)tid;
        s_sel[1] = less + excl;
        s_sel[2] = kr - excl;
      }
      __syncthreads();
      if (!take_all) {
        prefix = s_sel[0];
        less = s_sel[1];
        kr = s_sel[2];
      }
      __syncthreads();
    }
    if (take_all) break;
    if (use_cand && r < 7) {  // keep candidates whose top 8(r+1) bits equal the prefix
      const int nb = cb ^ 1;
      if (tid == 0) s_ncand[nb] = 0;
      __syncthreads();
      for (int64_t base = 0; base < scan_n; base += kThreads) {
        const int64_t i = base + tid;
        bool keep = false;
        uint16_t idx = 0;
        if (i < scan_n) {
          idx = cand[cb][i];
          keep = (key_at(idx) >> shift) == prefix;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        int off = 0;
        if ((tid & 31) == 0 && bal) off = atomicAdd(&s_ncand[nb], __popc(bal));
        off = __shfl_sync(0xffffffffu, off, 0);
        if (keep) cand[nb][off + __popc(bal & lanemask_lt())] = idx;
      }
      __syncthreads();
      cb = nb;
    }
  }
  const uint64_t T = take_all ? kInf : prefix;           // every evictable key < kInf
  const unsigned long long need_eq = take_all ? 0 : kr;  // keys == T to take, id order
  const unsigned long long n_sel = take_all ? total_ev : (unsigned long long)k;

  stamp();
  // ---------------- 2. order-preserving compaction (block-id order) ----------------
  // Blocked arrangement: thread t owns the contiguous slice range [t*ept, (t+1)*ept), so one
  // block scan of packed (eq << 16 | less) counts ranks every element in id order; equal
  // keys are taken in id order until the grid-wide quota need_eq is met.
  const int ept = (int)((cnt + kThreads - 1) / kThreads);
  const int64_t e0 = std::min<int64_t>(cnt, (int64_t)tid * ept), e1 = std::min<int64_t>(cnt, e0 + ept);
  int my_less = 0, my_eq = 0;
  for (int64_t i = e0; i < e1; ++i) {
    const uint64_t x = key_at(i);
    if (x == kInf) continue;
    my_less += x < T;
    my_eq += x == T;
  }
  long long tot_pk;
  const long long pk = block_excl_scan<long long>(((long long)my_eq << 32) | my_less, s_warp64, tot_pk);
  const long long tot_less = tot_pk & 0xFFFFFFFFll, tot_eq = tot_pk >> 32;
  if (tid == 0) sw->cnt_eq[c] = tot_eq;
  grid.sync();
  unsigned long long a = 0;
  for (int j = tid; j < c; j += kThreads) a += sw->cnt_eq[j];
  const unsigned long long eq_before = block_sum(a, s_red);
  const unsigned long long quota = eq_before >= need_eq ? 0ull : need_eq - eq_before;  // eq keys this CTA may take
  const unsigned long long eq_take = std::min<unsigned long long>((unsigned long long)tot_eq, quota);
  if (tid == 0) sw->cnt_sel[c] = (unsigned long long)tot_less + eq_take;
  grid.sync();
  a = 0;
  for (int j = tid; j < c; j += kThreads) a += sw->cnt_sel[j];
  const unsigned long long sel_before = block_sum(a, s_red);
  uint64_t loc_or = 0, loc_and_inv = 0;
  {
    unsigned long long less_r = (unsigned long long)(pk & 0xFFFFFFFFll), eq_r = (unsigned long long)(pk >> 32);
    for (int64_t i = e0; i < e1; ++i) {
      const uint64_t x = key_at(i);
      if (x == kInf) continue;
      const bool is_eq = x == T;
      if (x < T || (is_eq && eq_r < quota)) {
        const unsigned long long pos = sel_before + less_r + std::min(eq_r, quota);
        pk0[pos] = x;
        pi0[pos] = (int32_t)(lo + i);
        loc_or |= x;
        loc_and_inv |= ~x;
      }
      less_r += x < T;
      eq_r += is_eq;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    loc_or |= __shfl_xor_sync(0xffffffffu, loc_or, o);
    loc_and_inv |= __shfl_xor_sync(0xffffffffu, loc_and_inv, o);
  }
  if ((tid & 31) == 0 && (loc_or | loc_and_inv)) {
    atomicOr(&sw->key_or, (unsigned long long)loc_or);
    atomicOr(&sw->key_and_inv, (unsigned long long)loc_and_inv);
  }
  if (c == 0 && tid == 0) *d_count = (int64_t)n_sel;
  grid.sync();
  const uint64_t vary = sw->key_or & sw->key_and_inv;  // bits that differ among selected keys

  stamp();
  // ---------------- 3. stable LSD radix sort of (key, id) by key ----------------
  // S = min(#CTAs, ceil(m / kThreads)) sorter CTAs own contiguous ranges (one element per
  // thread for k = 64k).  Per 8-bit pass over the varying bytes only: (A) each sorter's digit
  // histogram -> global; grid barrier; (B) digit bases = digits below (all sorters) + same
  // digit in earlier sorters, then a stable scatter chunk by chunk (warp match_any ranks +
  // exclusive per-warp digit prefix); grid barrier ends the pass.
  uint64_t *ka = pk0, *kb = pk1;
  int32_t *ia = pi0, *ib = pi1;
  const int64_t m = (int64_t)n_sel;
  const int S = (int)std::min<int64_t>(C, std::max<int64_t>(1, (m + kThreads - 1) / kThreads));
  const int64_t sper = (m + S - 1) / S;
  const bool sorter = c < S;
  const int64_t slo = sorter ? std::min<int64_t>(m, c * sper) : 0;
  const int64_t shi = sorter ? std::min<int64_t>(m, slo + sper) : 0;
  const int w = tid >> 5;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 8 * pass;
    if (((vary >> shift) & 0xFF) == 0) continue;
    if (sorter) {
      for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
      __syncthreads();
      for (int64_t base = slo; base < shi; base += kThreads) {
        const int64_t i = base + tid;
        hist_add_fast(s_hist, i < shi ? (int)((ka[i] >> shift) & 0xFF) : 256);
      }
      __syncthreads();
      for (int i = tid; i < 256; i += kThreads) so->hist[c][i] = s_hist[i];
    }
    grid.sync();
    if (sorter) {
      unsigned int tot = 0, earlier = 0;
      if (tid < 256) {
#pragma unroll 16
        for (int j = 0; j < S; ++j) {
          const unsigned int h = so->hist[j][tid];
          tot += h;
          earlier += j < c ? h : 0u;
        }
      }
      int all;
      const int below = block_excl_scan(tid < 256 ? (int)tot : 0, s_warp, all);
      if (tid < 256) s_base[tid] = (unsigned int)below + earlier;
      __syncthreads();
      for (int64_t base = slo; base < shi; base += kThreads) {
        const int64_t i = base + tid;
        const bool have = i < shi;
        const uint64_t x = have ? ka[i] : 0;
        const int32_t xid = have ? ia[i] : 0;
        const int dg = have ? (int)((x >> shift) & 0xFF) : 256;
        uint4 *z = reinterpret_cast<uint4 *>(&s_wcnt[0][0]);
        for (int e = tid; e < kWarps * 256 / 4; e += kThreads) z[e] = make_uint4(0, 0, 0, 0);
        __syncthreads();
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const int wr = __popc(peers & lanemask_lt());
        if (dg < 256 && wr == 0) s_wcnt[w][dg] = __popc(peers);
        __syncthreads();
        for (int d = tid; d < 256; d += kThreads) {  // exclusive prefix over warps per digit
          unsigned int acc = 0;
          for (int ww = 0; ww < kWarps; ++ww) {
            const unsigned int v = s_wcnt[ww][d];
            s_wcnt[ww][d] = acc;
            acc += v;
          }
        }
        __syncthreads();
        if (have) {
          const unsigned int pos = s_base[dg] + s_wcnt[w][dg] + wr;
          kb[pos] = x;
          ib[pos] = xid;
        }
        __syncthreads();
        if (have && wr == 0) atomicAdd(&s_base[dg], (unsigned)__popc(peers));  // next chunk
        __syncthreads();
      }
    }
    grid.sync();
    stamp();
    uint64_t *tk = ka; ka = kb; kb = tk;
    int32_t *ti = ia; ia = ib; ib = ti;
  }
  for (int64_t i = (int64_t)c * kThreads + tid; i < m; i += (int64_t)C * kThreads) out_ids[i] = ia[i];
}

__global__ void free_ids_kernel(uint32_t *free_bits, const int32_t *ids, const int64_t *d_count,
                                int64_t k) {
  const int64_t n = min(*d_count, k);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t id = ids[i];
    atomicOr(free_bits + (id >> 5), 1u << (id & 31));
  }
}

struct ReleaseIds {
  int32_t n;
  int32_t ids[kReleaseBatch];
};
__global__ void release_ids_kernel(uint32_t *free_bits, const __grid_constant__ ReleaseIds r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x)
    atomicOr(free_bits + (r.ids[i] >> 5), 1u << (r.ids[i] & 31));
}

cudaError_t launch_release_ids(uint32_t *free_bits, const int32_t *ids_host, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  ReleaseIds r;
  r.n = n;
  std::memcpy(r.ids, ids_host, sizeof(int32_t) * n);
  release_ids_kernel<<<(n + 255) / 256, 256, 0, s>>>(free_bits, r);
  return cudaGetLastError();
}

cudaError_t launch_free_ids(uint32_t *free_bits, const int32_t *ids, const int64_t *d_count,
                            int64_t k, cudaStream_t s) {
  if (k <= 0) return cudaSuccess;
  free_ids_kernel<<<(unsigned)std::min<int64_t>((k + 255) / 256, 1184), 256, 0, s>>>(free_bits, ids, d_count, k);
  return cudaGetLastError();
}

cudaError_t launch_evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                int64_t *d_count, void *ws, size_t ws_bytes, cudaStream_t s) {
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // half the SMs: the selection is latency-bound, and runs concurrently with the attention
  // kernels (whose CTAs take the other SMs / share these)
  int C = std::max(1, std::min(nsm / 2, kMaxCtas));
  if (const char *e = getenv("KVA_EVICT_CTAS")) C = std::max(1, std::min(atoi(e), C));
  const int64_t per = (n + C - 1) / C;
  const size_t static_smem = 2 * 256 * 4 + 32 * 4 + 2 * 32 * 8 + 4 * 8 + kWarps * 256 * 4 + 1024;
  size_t dyn = (size_t)per * sizeof(uint64_t) + (per <= kCandCap ? 2 * (size_t)per * sizeof(uint16_t) : 0);
  int cache = 1;
  if (dyn + static_smem > (size_t)max_smem) { dyn = 0; cache = 0; }
  cudaError_t e = cudaFuncSetAttribute(evict_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  if (e != cudaSuccess) return e;
  // full shared-memory carveout so CTAs of concurrently running kernels can share an SM
  e = cudaFuncSetAttribute(evict_select_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e != cudaSuccess) return e;
  uint8_t *p = reinterpret_cast<uint8_t *>(ws);
  SelWs *sw = reinterpret_cast<SelWs *>(p);
  p += sizeof(SelWs);
  SortWs *so = reinterpret_cast<SortWs *>(p);
  p += sizeof(SortWs);
  const size_t pairs = (size_t)std::max<int64_t>(k, 1);
  uint64_t *pk0 = reinterpret_cast<uint64_t *>(p); p += pairs * 8;
  uint64_t *pk1 = reinterpret_cast<uint64_t *>(p); p += pairs * 8;
  int32_t *pi0 = reinterpret_cast<int32_t *>(p); p += pairs * 4;
  int32_t *pi1 = reinterpret_cast<int32_t *>(p); p += pairs * 4;
  if ((size_t)(p - reinterpret_cast<uint8_t *>(ws)) > ws_bytes) return cudaErrorInvalidValue;
  e = cudaMemsetAsync(sw, 0, sizeof(SelWs), s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&keys, (void *)&n, (void *)&k, (void *)&out_ids, (void *)&d_count,
                  (void *)&sw, (void *)&so, (void *)&pk0, (void *)&pi0, (void *)&pk1, (void *)&pi1,
                  (void *)&cache};
  return cudaLaunchCooperativeKernel((void *)evict_select_kernel, dim3(C), dim3(kThreads), args, dyn, s);
}

}  // namespace kva
