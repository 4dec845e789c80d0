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
constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCtas = 1024;

struct SelWs {  // global scratch (zeroed by the host before launch)
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

// Block-wide exclusive scan of one int per thread; `total` gets the block sum.
__device__ __forceinline__ int block_excl_scan(int v, int *s_warp, int &total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = lane < kWarps ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_warp[lane] = t;  // inclusive prefix over warps
  }
  __syncthreads();
  total = s_warp[kWarps - 1];
  const int res = x - v + (w > 0 ? s_warp[w - 1] : 0);
  __syncthreads();
  return res;
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

__global__ void __launch_bounds__(kThreads, 1)
    evict_select_kernel(const uint64_t *__restrict__ keys, int64_t n, int64_t k,
                        int32_t *__restrict__ out_ids, int64_t *__restrict__ d_count,
                        SelWs *__restrict__ sw, SortWs *__restrict__ so, uint64_t *pk0,
                        int32_t *pi0, uint64_t *pk1, int32_t *pi1, int cache_keys) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint64_t s_keys[];
  __shared__ unsigned int s_hist[256];
  __shared__ unsigned int s_base[256];
  __shared__ int s_warp[32];
  __shared__ unsigned long long s_red[32];
  __shared__ unsigned long long s_sel[4];
  __shared__ unsigned int s_wcnt[kWarps][256];  // 32 KB
  const int C = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const int64_t per = (n + C - 1) / C;
  const int64_t lo = std::min<int64_t>(n, c * per), hi = std::min<int64_t>(n, lo + per);
  const int64_t cnt = hi - lo;
  if (cache_keys)
    for (int64_t i = tid; i < cnt; i += kThreads) s_keys[i] = keys[lo + i];
  __syncthreads();
  auto key_at = [&](int64_t i) -> uint64_t { return cache_keys ? s_keys[i] : keys[lo + i]; };

  // ---------------- 1. radix select: T = k-th smallest evictable key ----------------
  uint64_t prefix = 0;
  unsigned long long kr = (unsigned long long)k, less = 0, total_ev = 0;
  bool take_all = false;
  for (int r = 0; r < 8; ++r) {
    const int shift = 56 - 8 * r;
    for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    for (int64_t i = tid; i < cnt; i += kThreads) {
      const uint64_t x = key_at(i);
      if (x == kInf) continue;
      if (r > 0 && (x >> (shift + 8)) != prefix) continue;
      atomicAdd(&s_hist[(x >> shift) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = tid; i < 256; i += kThreads)
      if (s_hist[i]) atomicAdd(&sw->hist[r][i], (unsigned long long)s_hist[i]);
    grid.sync();
    if (tid == 0) {
      if (r == 0) {
        for (int i = 0; i < 256; ++i) total_ev += sw->hist[0][i];
        take_all = total_ev <= kr;
      }
      if (!take_all) {
        unsigned long long acc = 0;
        int dsel = 255;
        for (int i = 0; i < 256; ++i) {
          const unsigned long long h = sw->hist[r][i];
          if (acc + h >= kr) { dsel = i; break; }
          acc += h;
        }
        kr -= acc;
        less += acc;
        prefix = (prefix << 8) | (uint64_t)dsel;
      }
      s_sel[0] = prefix;
      s_sel[1] = less;
      s_sel[2] = kr;
      s_sel[3] = total_ev | (take_all ? (1ull << 63) : 0ull);
    }
    __syncthreads();
    prefix = s_sel[0];
    less = s_sel[1];
    kr = s_sel[2];
    total_ev = s_sel[3] & ~(1ull << 63);
    take_all = (s_sel[3] >> 63) != 0;
    __syncthreads();
    if (take_all) break;
  }
  const uint64_t T = take_all ? kInf : prefix;           // every evictable key < kInf
  const unsigned long long need_eq = take_all ? 0 : kr;  // keys == T to take, id order
  const unsigned long long n_sel = take_all ? total_ev : (unsigned long long)k;

  // ---------------- 2. order-preserving compaction (block-id order) ----------------
  int my_less = 0, my_eq = 0;
  for (int64_t i = tid; i < cnt; i += kThreads) {
    const uint64_t x = key_at(i);
    if (x == kInf) continue;
    my_less += x < T;
    my_eq += x == T;
  }
  int tot_less, tot_eq;
  block_excl_scan(my_less, s_warp, tot_less);
  block_excl_scan(my_eq, s_warp, tot_eq);
  if (tid == 0) sw->cnt_eq[c] = tot_eq;
  grid.sync();
  unsigned long long a = 0;
  for (int j = tid; j < c; j += kThreads) a += sw->cnt_eq[j];
  const unsigned long long eq_before = block_sum(a, s_red);
  const unsigned long long eq_take =
      eq_before >= need_eq ? 0ull : std::min<unsigned long long>((unsigned long long)tot_eq, need_eq - eq_before);
  if (tid == 0) sw->cnt_sel[c] = (unsigned long long)tot_less + eq_take;
  grid.sync();
  a = 0;
  for (int j = tid; j < c; j += kThreads) a += sw->cnt_sel[j];
  const unsigned long long sel_before = block_sum(a, s_red);
  unsigned long long run_sel = 0, run_eq = 0;
  uint64_t loc_or = 0, loc_and_inv = 0;
  for (int64_t base = 0; base < cnt; base += kThreads) {
    const int64_t i = base + tid;
    const uint64_t x = i < cnt ? key_at(i) : kInf;
    const int is_eq = (x != kInf && x == T) ? 1 : 0;
    int eq_tot;
    const int eq_rank = block_excl_scan(is_eq, s_warp, eq_tot);
    const bool sel = (x != kInf) && (x < T || (is_eq && eq_before + run_eq + eq_rank < need_eq));
    int sel_tot;
    const int sel_rank = block_excl_scan(sel ? 1 : 0, s_warp, sel_tot);
    if (sel) {
      const unsigned long long pos = sel_before + run_sel + sel_rank;
      pk0[pos] = x;
      pi0[pos] = (int32_t)(lo + i);
      loc_or |= x;
      loc_and_inv |= ~x;
    }
    run_sel += sel_tot;
    run_eq += eq_tot;
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

  // ---------------- 3. stable LSD radix sort of (key, id) by key ----------------
  uint64_t *ka = pk0, *kb = pk1;
  int32_t *ia = pi0, *ib = pi1;
  const int64_t m = (int64_t)n_sel;
  const int64_t sper = (m + C - 1) / C;
  const int64_t slo = std::min<int64_t>(m, c * sper), shi = std::min<int64_t>(m, slo + sper);
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 8 * pass;
    if (((vary >> shift) & 0xFF) == 0) continue;
    for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    for (int64_t i = slo + tid; i < shi; i += kThreads) atomicAdd(&s_hist[(ka[i] >> shift) & 0xFF], 1u);
    __syncthreads();
    for (int i = tid; i < 256; i += kThreads) so->hist[c][i] = s_hist[i];
    grid.sync();
    // base[d] = #elements with digit < d (all CTAs) + #elements with digit d in CTAs < c
    {
      const int d = tid < 256 ? tid : 0;
      unsigned int tot = 0, earlier = 0;
      if (tid < 256)
        for (int j = 0; j < C; ++j) {
          const unsigned int h = so->hist[j][d];
          tot += h;
          earlier += j < c ? h : 0u;
        }
      int all;
      const int below = block_excl_scan(tid < 256 ? (int)tot : 0, s_warp, all);
      if (tid < 256) s_base[d] = (unsigned int)below + earlier;
      __syncthreads();
    }
    for (int64_t base = slo; base < shi; base += kThreads) {
      const int64_t i = base + tid;
      const bool valid = i < shi;
      const uint64_t x = valid ? ka[i] : 0;
      const int dg = valid ? (int)((x >> shift) & 0xFF) : 256;
      const int w = tid >> 5;
      for (int e = tid; e < kWarps * 256; e += kThreads) (&s_wcnt[0][0])[e] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      const int wr = __popc(peers & lanemask_lt());
      if (valid && wr == 0) s_wcnt[w][dg] = __popc(peers);
      __syncthreads();
      if (tid < 256) {  // exclusive prefix over warps, per digit
        unsigned int acc = 0;
        for (int ww = 0; ww < kWarps; ++ww) {
          const unsigned int v = s_wcnt[ww][tid];
          s_wcnt[ww][tid] = acc;
          acc += v;
        }
      }
      __syncthreads();
      if (valid) {
        const unsigned int pos = s_base[dg] + s_wcnt[w][dg] + wr;
        kb[pos] = x;
        ib[pos] = ia[i];
      }
      __syncthreads();
      if (valid) atomicAdd(&s_base[dg], 1u);  // advance bases by this chunk's counts
      __syncthreads();
    }
    grid.sync();
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
  const int C = std::max(1, std::min(nsm, kMaxCtas));
  const int64_t per = (n + C - 1) / C;
  const size_t static_smem = 2 * 256 * 4 + 32 * 4 + 32 * 8 + 4 * 8 + kWarps * 256 * 4 + 1024;
  size_t dyn = (size_t)per * sizeof(uint64_t);
  int cache = 1;
  if (dyn + static_smem > (size_t)max_smem) { dyn = 0; cache = 0; }
  cudaError_t e = cudaFuncSetAttribute(evict_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
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
