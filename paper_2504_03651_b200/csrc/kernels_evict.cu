// kernels_evict.cu — task-aware eviction: priority keys and the radix
// top-k that replaces the paper's host-side free-table priority queue.
//
// Order: "When evicting the KV cache, we will first consider the priority of the KV cache
// entry, and then the last access time"; priorities P:331-334.  Keys are
// order-preserving u64 codes (readings #18-#20); equal keys are broken by block id.
//
// evict_select is one cooperative persistent kernel (grid = #SMs / 2, 512 threads, keys of a
// CTA's slice cached in shared memory):
//   1. MSD radix select over 8-bit digits (only bytes that vary among the evictable keys, and
//      only until the chosen bin is taken whole) -> threshold prefix P at bit level lvl and
//      count(key >> lvl < P);
//   2. order-preserving compaction of {key >> lvl < P} u {first quota blocks with
//      key >> lvl == P} (block-id order) into a (key, id) array;
//   3. stable LSD radix sort of that array by key over only the bytes that vary (stability
//      keeps block-id order among equal keys), one grid barrier per pass.
// Grid-wide steps are separated by cooperative-groups grid barriers (select rounds + 2 + passes).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

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
// KV-manager step.  Transitions arrive as the caller's raw chains (host
// validated, uploaded unchanged); "last chain wins" is resolved on the device: every listed
// block's winner slot is reset, then takes the max element index listing it (atomicMax), and
// only that element applies its chain's state.  Then the reference counts (recount: zeroed
// by the host + atomicAdd; incremental: atomicAdd / atomicSub), then keys + active count.
__global__ void manager_win_init_kernel(const int32_t *__restrict__ tr_ids, int64_t n_tr, int32_t *__restrict__ win,
                                        unsigned long long *__restrict__ n_active) {
  if (n_active && blockIdx.x == 0 && threadIdx.x == 0) *n_active = 0ull;  // counted by the keys kernel
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_tr; e += (int64_t)gridDim.x * blockDim.x)
    win[tr_ids[e]] = -1;
}
__global__ void manager_win_max_kernel(const int32_t *__restrict__ tr_ids, int64_t n_tr, int32_t *__restrict__ win) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_tr; e += (int64_t)gridDim.x * blockDim.x)
    atomicMax(&win[tr_ids[e]], (int32_t)e);
}

__global__ void manager_apply_kernel(uint8_t *__restrict__ state, uint32_t *__restrict__ rc,
                                     uint32_t *__restrict__ lat, int64_t n, uint32_t now,
                                     const int32_t *__restrict__ tr_ids, int64_t n_tr,
                                     const int32_t *__restrict__ tr_indptr, const uint8_t *__restrict__ tr_state,
                                     int32_t n_chains, const int32_t *__restrict__ win,
                                     const int32_t *__restrict__ pool_ids, int64_t pool_len,
                                     const int32_t *__restrict__ del_ids, int64_t del_len) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_tr + pool_len + del_len;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (e < n_tr) {
      const int32_t id = tr_ids[e];  // validated on the host
      if (win[id] != (int32_t)e) continue;  // a later chain lists this block too
      int lo = 0, hi = n_chains - 1;       // chain j: indptr[j] <= e < indptr[j + 1]
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tr_indptr[mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      state[id] = tr_state[lo];
      lat[id] = now;
    } else if (e < n_tr + pool_len) {
      const int32_t id = pool_ids[e - n_tr];
      if ((uint64_t)id < (uint64_t)n) atomicAdd(&rc[id], 1u);
    } else {
      const int32_t id = del_ids[e - n_tr - pool_len];
      if ((uint64_t)id < (uint64_t)n) atomicSub(&rc[id], 1u);
    }
  }
}

__global__ void manager_keys_kernel(const uint8_t *__restrict__ state, const uint32_t *__restrict__ rc,
                                    const uint32_t *__restrict__ lat, const uint16_t *__restrict__ depth,
                                    int64_t n, uint64_t *__restrict__ keys,
                                    unsigned long long *__restrict__ n_active) {
  unsigned int act = 0;
  auto one = [&](uint32_t s, uint32_t r, uint32_t la, uint32_t dp) -> uint64_t {
    act += (s == 1 || s == 2 || (s >= 3 && s <= 5 && r > 0)) ? 1u : 0u;
    if (s == 0 || s == 1 || s == 2 || s > 5) return kInf;
    uint64_t code;
    if (r > 0) code = r >= 0x7FFFu ? 0xFFFEull : 2ull * r;
    else code = (s == 4) ? 1ull : 0ull;
    return (code << 48) | ((uint64_t)la << 16) | (0xFFFFull - (uint64_t)dp);
  };
  // 4 blocks per thread with vector loads/stores when the arrays allow it (torch allocations
  // are 256-B aligned), scalar tail
  const bool vec = ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(rc) |
                     reinterpret_cast<uintptr_t>(lat) | reinterpret_cast<uintptr_t>(keys) |
                     (depth ? reinterpret_cast<uintptr_t>(depth) : 0)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t s4 = reinterpret_cast<const uint32_t *>(state)[q];
    const uint4 r4 = reinterpret_cast<const uint4 *>(rc)[q];
    const uint4 l4 = reinterpret_cast<const uint4 *>(lat)[q];
    uint2 d4 = make_uint2(0u, 0u);
    if (depth) d4 = reinterpret_cast<const uint2 *>(depth)[q];
    const uint64_t k0 = one(s4 & 0xFF, r4.x, l4.x, d4.x & 0xFFFF);
    const uint64_t k1 = one((s4 >> 8) & 0xFF, r4.y, l4.y, d4.x >> 16);
    const uint64_t k2 = one((s4 >> 16) & 0xFF, r4.z, l4.z, d4.y & 0xFFFF);
    const uint64_t k3 = one(s4 >> 24, r4.w, l4.w, d4.y >> 16);
    reinterpret_cast<ulonglong2 *>(keys)[2 * q] = make_ulonglong2(k0, k1);
    reinterpret_cast<ulonglong2 *>(keys)[2 * q + 1] = make_ulonglong2(k2, k3);
  }
  for (int64_t b = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < n;
       b += (int64_t)gridDim.x * blockDim.x)
    keys[b] = one(state[b], rc[b], lat[b], depth ? depth[b] : 0u);
  if (n_active) {  // one atomic per CTA (a per-warp atomic on one address serialises in L2)
    __shared__ unsigned int s_act;
    if (threadIdx.x == 0) s_act = 0u;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) act += __shfl_xor_sync(0xffffffffu, act, o);
    if ((threadIdx.x & 31) == 0 && act) atomicAdd(&s_act, act);
    __syncthreads();
    if (threadIdx.x == 0 && s_act) atomicAdd(n_active, (unsigned long long)s_act);
  }
}

cudaError_t launch_manager_step(uint8_t *state, uint32_t *rc, uint32_t *lat, const uint16_t *depth,
                                int64_t n, uint32_t now, const int32_t *tr_ids, int64_t n_tr,
                                const int32_t *tr_indptr, const uint8_t *tr_state, int32_t n_chains,
                                int32_t *win, bool recount, const int32_t *pool_ids, int64_t pool_len,
                                const int32_t *del_ids, int64_t del_len, uint64_t *keys, int64_t *n_active,
                                cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  if (recount) e = cudaMemsetAsync(rc, 0, (size_t)n * sizeof(uint32_t), s);
  // the active count is zeroed by the winner-init kernel when there are transitions
  if (e == cudaSuccess && n_active && n_tr <= 0) e = cudaMemsetAsync(n_active, 0, sizeof(int64_t), s);
  if (e != cudaSuccess) return e;
  auto grid_for = [](int64_t m) { return (int)std::min<int64_t>((m + 255) / 256, 148 * 8); };
  if (n_tr > 0) {
    manager_win_init_kernel<<<grid_for(n_tr), 256, 0, s>>>(tr_ids, n_tr, win,
                                                           reinterpret_cast<unsigned long long *>(n_active));
    manager_win_max_kernel<<<grid_for(n_tr), 256, 0, s>>>(tr_ids, n_tr, win);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  const int64_t m = n_tr + pool_len + del_len;
  if (m > 0) {
    manager_apply_kernel<<<grid_for(m), 256, 0, s>>>(state, rc, lat, n, now, tr_ids, n_tr, tr_indptr, tr_state,
                                                     n_chains, win, pool_ids, pool_len, del_ids, del_len);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (n > 0) {
    manager_keys_kernel<<<grid_for(n), 256, 0, s>>>(state, rc, lat, depth, n, keys,
                                                    reinterpret_cast<unsigned long long *>(n_active));
    e = cudaGetLastError();
  }
  return e;
}

// ---------------------------------------------------------------------------------------
namespace {
constexpr int kThreads = 512;  // leaves registers/smem for a co-resident decode CTA
constexpr int kWarps = kThreads / 32;
constexpr int kMaxCtas = kThreads;  // the compaction scans one value per CTA block-wide

struct SelWs {  // global scratch (zeroed by the host before launch)
  unsigned long long t[32];      // phase timestamps of CTA 0 (%globaltimer, ns; diagnostics)
  unsigned long long hist[8][256];
  unsigned long long cnt[kMaxCtas];           // per CTA: (#eq << 32) | #less
  unsigned long long ev_or, ev_and_inv;       // OR of evictable keys, OR of their complements
  unsigned long long key_or, key_and_inv;     // same over the selected keys
};
struct SortWs {
  // digit counts of one LSD pass, [sorter CTA][digit] (a warp reading 32 digits of one sorter
  // row is one coalesced 128-B access), triple-buffered: pass p reads buffer p%3, its scatter accumulates pass p+1's counts into
  // buffer (p+1)%3, and buffer (p+2)%3 (last read in pass p-1) is zeroed
  unsigned int hist[3][256 * kMaxCtas];
};
}  // namespace

// ---------------------------------------------------------------------------------------
// Sample-bucket path of evict_select (KVA_EVICT_IMPL=fast, n >= 2^16): sample -> splitters -> one bucketing pass
// -> per-bucket sorts.  Three launches, no grid barrier; the exact cooperative kernel above is
// the fallback (it runs only if a bucket overflows or the sample under-estimated the k-th key).
//   1. one CTA sorts a strided sample of kSample (2048) keys and picks v_hi = the sample element at
//      rank r + 4 sqrt(r) + 8 (r = k * kSample / n) and kBuckets - 1 splitters below it;
//   2. every key < v_hi goes to its bucket (key range), positions reserved per CTA tile;
//   3. bucket b's CTA checks that the candidates hold >= k keys (then they contain every key
//      <= the k-th smallest, ties included), sorts its bucket by (key, id) in shared memory and
//      writes the ranks < k of the global order.
namespace {
constexpr int kSample = 2048;
constexpr int kBuckets = 64;
constexpr int kCap = 8192;  // pairs per bucket (its shared-memory sort: 8192 x 12 B)
struct FastWs {
  unsigned long long split[kBuckets];  // split[b] = first key of bucket b + 1 (b < kBuckets - 1)
  unsigned long long v_hi;             // candidates: key < v_hi (UINT64_MAX: every evictable key)
  unsigned int cnt[kBuckets];
  int overflow;
  int run_fallback;
};
}  // namespace

__device__ __forceinline__ bool pair_gt(uint64_t ka, int32_t ia, uint64_t kb, int32_t ib) {
  return ka > kb || (ka == kb && ia > ib);
}

// bitonic sort of N (power of two) (key, id) pairs in shared memory, ascending
__device__ void smem_bitonic(uint64_t *k, int32_t *id, int N) {
  for (int size = 2; size <= N; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          if (pair_gt(k[i], id[i], k[j], id[j]) == up) {
            const uint64_t tk = k[i]; k[i] = k[j]; k[j] = tk;
            const int32_t ti = id[i]; id[i] = id[j]; id[j] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(1024) sel_sample_kernel(const uint64_t *__restrict__ keys, int64_t n,
                                                          int64_t k, FastWs *__restrict__ fw) {
  __shared__ uint64_t sk[kSample];
  __shared__ int32_t si[kSample];
  __shared__ int s_ev;
  const int tid = threadIdx.x;
  if (tid < kBuckets) fw->cnt[tid] = 0u;
  if (tid == 0) {
    fw->overflow = 0;
    fw->run_fallback = 0;
    s_ev = 0;
  }
  __syncthreads();
  int ev = 0;
  for (int i = tid; i < kSample; i += blockDim.x) {
    const uint64_t key = keys[(int64_t)(((__int128)i * n) / kSample)];
    sk[i] = key;
    si[i] = i;
    ev += key != kInf;
  }
  atomicAdd(&s_ev, ev);
  __syncthreads();
  smem_bitonic(sk, si, kSample);
  if (tid == 0) {
    const double r = (double)k * kSample / (double)n;
    const int64_t r_hi = (int64_t)ceil(r + 4.0 * sqrt(r) + 8.0);
    const int evs = s_ev;
    int top;  // sample ranks [0, top) are spread over the buckets
    if (r_hi >= evs) {
      fw->v_hi = kInf;  // the candidates may have to be every evictable key
      top = evs;
    } else {
      fw->v_hi = sk[r_hi];
      top = (int)r_hi;
    }
    for (int b = 0; b < kBuckets - 1; ++b) {
      const int rk = (int)(((int64_t)top * (b + 1)) / kBuckets);
      fw->split[b] = top > 0 ? sk[min(rk, kSample - 1)] : kInf;
    }
  }
}

__global__ void __launch_bounds__(256) sel_bucket_kernel(const uint64_t *__restrict__ keys, int64_t n,
                                                         FastWs *__restrict__ fw, uint64_t *__restrict__ bkey,
                                                         int32_t *__restrict__ bid) {
  constexpr int PER = 16;  // keys per thread per tile
  __shared__ uint64_t s_split[kBuckets];
  __shared__ unsigned int s_cnt[kBuckets], s_base[kBuckets];
  const int tid = threadIdx.x;
  if (tid < kBuckets) s_split[tid] = fw->split[tid];
  __syncthreads();
  const uint64_t v_hi = fw->v_hi;
  const int64_t tile = (int64_t)blockDim.x * PER;
  for (int64_t t0 = (int64_t)blockIdx.x * tile; t0 < n; t0 += (int64_t)gridDim.x * tile) {
    if (tid < kBuckets) s_cnt[tid] = 0u;
    __syncthreads();
    int8_t bk[PER];
    unsigned int lp[PER];
    uint64_t kv[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int64_t i = t0 + (int64_t)u * blockDim.x + tid;  // coalesced
      bk[u] = -1;
      if (i < n) {
        const uint64_t key = keys[i];
        kv[u] = key;
        if (key < v_hi && key != kInf) {
          int lo = 0, hi = kBuckets - 1;  // bucket = #splitters <= key
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s_split[mid] <= key) lo = mid + 1;
            else hi = mid;
          }
          bk[u] = (int8_t)lo;
          lp[u] = atomicAdd(&s_cnt[lo], 1u);
        }
      }
    }
    __syncthreads();
    if (tid < kBuckets) s_base[tid] = s_cnt[tid] ? atomicAdd(&fw->cnt[tid], s_cnt[tid]) : 0u;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (bk[u] < 0) continue;
      const unsigned int pos = s_base[bk[u]] + lp[u];
      if (pos < (unsigned)kCap) {
        bkey[(int64_t)bk[u] * kCap + pos] = kv[u];
        bid[(int64_t)bk[u] * kCap + pos] = (int32_t)(t0 + (int64_t)u * blockDim.x + tid);
      } else {
        fw->overflow = 1;
      }
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) sel_sort_kernel(int64_t k, FastWs *__restrict__ fw,
                                                        const uint64_t *__restrict__ bkey,
                                                        const int32_t *__restrict__ bid,
                                                        int32_t *__restrict__ out_ids, int64_t *__restrict__ d_count) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint64_t *sk = reinterpret_cast<uint64_t *>(sm);
  int32_t *si = reinterpret_cast<int32_t *>(sm + (size_t)kCap * 8);
  const int b = blockIdx.x, tid = threadIdx.x;
  int64_t total = 0, off = 0;
  for (int j = 0; j < kBuckets; ++j) {
    const int64_t c = fw->cnt[j];
    if (j < b) off += c;
    total += c;
  }
  const bool inf_mode = fw->v_hi == kInf;
  const bool valid = !fw->overflow && (inf_mode || total >= k);
  if (b == 0 && tid == 0) {
    fw->run_fallback = valid ? 0 : 1;
    if (valid) *d_count = total < k ? total : k;
  }
  const int64_t cnt = fw->cnt[b];
  if (!valid || off >= k || cnt == 0) return;
  int N = 2;
  while (N < cnt) N <<= 1;
  for (int i = tid; i < N; i += blockDim.x) {
    if (i < cnt) {
      sk[i] = bkey[(int64_t)b * kCap + i];
      si[i] = bid[(int64_t)b * kCap + i];
    } else {
      sk[i] = kInf;
      si[i] = INT32_MAX;
    }
  }
  __syncthreads();
  smem_bitonic(sk, si, N);
  for (int64_t i = tid; i < cnt && off + i < k; i += blockDim.x) out_ids[off + i] = si[i];
}

size_t evict_select_ws_bytes(int64_t n, int64_t k) {
  (void)n;
  const size_t pairs = (size_t)std::max<int64_t>(k, 1);
  return sizeof(SelWs) + sizeof(SortWs) + 2 * pairs * (sizeof(uint64_t) + sizeof(int32_t)) + 256 +
         ((sizeof(FastWs) + 255) & ~size_t(255)) + (size_t)kBuckets * kCap * (8 + 4) + 256;
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

__global__ void __launch_bounds__(kThreads, 2)
    evict_select_kernel(const uint64_t *__restrict__ keys, int64_t n, int64_t k,
                        int32_t *__restrict__ out_ids, int64_t *__restrict__ d_count,
                        SelWs *__restrict__ sw, SortWs *__restrict__ so, uint64_t *pk0,
                        int32_t *pi0, uint64_t *pk1, int32_t *pi1, int cache_keys,
                        const int *__restrict__ run_flag) {
  // fallback of the sample-bucket fast path: every CTA leaves before any grid barrier when the
  // fast path produced the result (run_flag == 0); run_flag == nullptr: always run
  if (run_flag && *(volatile const int *)run_flag == 0) return;
  cg::grid_group grid = cg::this_grid();
  int tp = 0;
  auto stamp = [&]() {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (tp < 32) sw->t[tp] = t;  // (a sorter when c == 0)
    }
    ++tp;
  };
  stamp();
  extern __shared__ __align__(16) uint64_t s_keys[];
  __shared__ unsigned int s_hist[256];
  __shared__ unsigned int s_base[256];
  __shared__ unsigned int s_part[256];
  __shared__ int s_warp[32];
  __shared__ long long s_warp64[32];
  __shared__ unsigned long long s_sel[4];
  __shared__ __align__(16) unsigned int s_wcnt[kWarps][256];  // 16 KB
  const int C = gridDim.x, c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t per = (((n + C - 1) / C) + 1) & ~1ll;  // even: 16-B aligned slices
  const int64_t lo = std::min<int64_t>(n, c * per), hi = std::min<int64_t>(n, lo + per);
  const int64_t cnt = hi - lo;
  auto key_at = [&](int64_t i) -> uint64_t { return cache_keys ? s_keys[i] : keys[lo + i]; };

  // ---------------- 0. slice -> shared memory (16-B vector loads, 8 in flight) ----------------
  if (cache_keys && (reinterpret_cast<uintptr_t>(keys) & 15)) {
    for (int64_t i = tid; i < cnt; i += kThreads) s_keys[i] = keys[lo + i];
  } else if (cache_keys) {
    const int64_t nv = cnt >> 1;
    const uint4 *src = reinterpret_cast<const uint4 *>(keys + lo);
    uint4 *dst = reinterpret_cast<uint4 *>(s_keys);
    for (int64_t b = 0; b < nv; b += 8 * kThreads) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = b + u * kThreads + tid;
        if (i < nv) v[u] = __ldg(src + i);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = b + u * kThreads + tid;
        if (i < nv) dst[i] = v[u];
      }
    }
    if ((cnt & 1) && tid == 0) s_keys[cnt - 1] = keys[lo + cnt - 1];
  }
  {
    uint4 *z = reinterpret_cast<uint4 *>(&s_wcnt[0][0]);
    for (int e = tid; e < kWarps * 256 / 4; e += kThreads) z[e] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();

  // Digit histogram of one select round over the whole slice: keys matching the current
  // prefix (bits above `shift + 8`) count their digit at `shift`.  Each thread keeps a
  // run-length counter flushed into its warp's private histogram; the warp histograms are
  // summed into the global one.  (Warp aggregation with match_any instead: slower, 7.2 vs
  // 5.9 us per round.)
  // Round 0 (`all`) also ORs the evictable keys and their complements (the bytes that vary
  // decide which later rounds run) in the same pass.
  auto round_hist = [&](int r, int shift, uint64_t prefix, bool all) -> void {
    constexpr int kU = 8;  // keys per thread in flight (L2 latency)
    int run_d = -1;
    unsigned run_n = 0;
    uint64_t lor = 0, linv = 0;
    for (int64_t base = 0; base < cnt; base += kU * kThreads) {
      uint64_t x[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = base + u * kThreads + tid;
        x[u] = i < cnt ? key_at(i) : kInf;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const bool match = x[u] != kInf && (all || (x[u] >> (shift + 8)) == prefix);
        const int d = match ? (int)((x[u] >> shift) & 0xFF) : -1;
        if (all && x[u] != kInf) {
          lor |= x[u];
          linv |= ~x[u];
        }
        if (d != run_d) {
          if (run_n) atomicAdd(&s_wcnt[w][run_d], run_n);
          run_d = d;
          run_n = 0;
        }
        run_n += d >= 0;
      }
    }
    if (run_n) atomicAdd(&s_wcnt[w][run_d], run_n);
    if (all) {
      for (int o = 16; o > 0; o >>= 1) {
        lor |= __shfl_xor_sync(0xffffffffu, lor, o);
        linv |= __shfl_xor_sync(0xffffffffu, linv, o);
      }
      if (lane == 0 && (lor | linv)) {
        atomicOr(&sw->ev_or, (unsigned long long)lor);
        atomicOr(&sw->ev_and_inv, (unsigned long long)linv);
      }
    }
    __syncthreads();
    for (int d = tid; d < 256; d += kThreads) {
      unsigned t = 0;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) {
        t += s_wcnt[ww][d];
        s_wcnt[ww][d] = 0;
      }
      if (t) atomicAdd(&sw->hist[r][d], (unsigned long long)t);
    }
  };

  round_hist(0, 56, 0, true);  // + OR / AND of the evictable keys
  stamp();  // 1: keys cached, round-0 histogram built

  // ---------------- 1. radix select: threshold prefix P at bit level lvl ----------------
  // MSD rounds of 8-bit digits; rounds whose byte is constant over the evictable keys are
  // skipped without a barrier; the select stops as soon as the chosen bin is taken whole or
  // no lower bit varies.  Selected = {key >> lvl < P} + the first need_eq (block-id order)
  // of {key >> lvl == P}.
  uint64_t prefix = 0, ev_or = 0, vary_ev = 0;
  unsigned long long kr = (unsigned long long)k, less = 0, total_ev = 0;
  bool take_all = false;
  int lvl = 56;
  for (int r = 0; r < 8; ++r) {
    const int shift = 56 - 8 * r;
    lvl = shift;
    if (r > 0) {
      if (((vary_ev >> shift) & 0xFF) == 0) {  // constant byte: every candidate has it
        prefix = (prefix << 8) | ((ev_or >> shift) & 0xFF);
        continue;
      }
      round_hist(r, shift, prefix, false);
    }
    stamp();
    grid.sync();
    stamp();
    if (r == 0) {
      ev_or = sw->ev_or;
      vary_ev = ev_or & sw->ev_and_inv;
    }
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
      s_sel[3] = (unsigned long long)h;
    }
    __syncthreads();
    if (take_all) break;
    prefix = s_sel[0];
    less = s_sel[1];
    kr = s_sel[2];
    const bool whole_bin = kr == s_sel[3];
    __syncthreads();
    if (whole_bin || (vary_ev & ((1ull << shift) - 1)) == 0) break;
  }
  if (take_all) {
    prefix = kInf;
    lvl = 0;
  }
  const uint64_t P = prefix;
  const unsigned long long need_eq = take_all ? 0 : kr;  // keys with key >> lvl == P to take
  const unsigned long long n_sel = take_all ? total_ev : (unsigned long long)k;

  stamp();
  // ---------------- 2. order-preserving compaction (block-id order) ----------------
  // Warp-blocked arrangement: warp w owns the contiguous slice range [w*wlen, (w+1)*wlen),
  // walked 32 keys at a time, so ballots rank every key in id order.  After one grid barrier
  // every CTA scans all CTAs' (less, eq) counts itself: keys with key >> lvl == P are taken in
  // id order until the grid-wide quota need_eq is met.
  const int64_t wlen = ((cnt + kThreads - 1) / kThreads) * 32;
  const int64_t w0 = std::min<int64_t>(cnt, (int64_t)w * wlen), w1 = std::min<int64_t>(cnt, w0 + wlen);
  const unsigned lt = lanemask_lt();
  // kW 32-key groups per warp in flight (L2 latency bound)
  constexpr int kW = 8;
  auto classify_x = [&](uint64_t x, bool &is_less, bool &is_eq) {
    const uint64_t xh = x >> lvl;
    is_less = x != kInf && xh < P;
    is_eq = x != kInf && xh == P;
  };
  unsigned my_less = 0, my_eq = 0;
  for (int64_t g0 = w0; g0 < w1; g0 += kW * 32) {
    uint64_t xs[kW];
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const int64_t i = g0 + u * 32 + lane;
      xs[u] = i < w1 ? key_at(i) : kInf;
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      bool l, e;
      classify_x(xs[u], l, e);
      my_less += __popc(__ballot_sync(0xffffffffu, l));
      my_eq += __popc(__ballot_sync(0xffffffffu, e));
    }
  }
  long long tot_pk;
  const long long pk = block_excl_scan<long long>(lane == 0 ? ((long long)my_eq << 32) | my_less : 0ll,
                                                  s_warp64, tot_pk);
  const long long wbase = __shfl_sync(0xffffffffu, pk, 0);  // this warp's (eq, less) base
  if (tid == 0) sw->cnt[c] = (unsigned long long)tot_pk;
  stamp();
  grid.sync();
  stamp();
  {
    const unsigned long long v = tid < C ? sw->cnt[tid] : 0ull;
    const long long eq_j = (long long)(v >> 32), less_j = (long long)(v & 0xFFFFFFFFull);
    long long t1, t2;
    const long long eq_before = block_excl_scan<long long>(eq_j, s_warp64, t1);
    const long long quota = (long long)need_eq > eq_before ? (long long)need_eq - eq_before : 0;
    const long long sel_j = less_j + std::min(eq_j, quota);
    const long long sel_before = block_excl_scan<long long>(sel_j, s_warp64, t2);
    if (tid == c) {
      s_sel[0] = (unsigned long long)sel_before;
      s_sel[1] = (unsigned long long)quota;
    }
    __syncthreads();
  }
  const unsigned long long sel_before = s_sel[0], quota = s_sel[1];
  uint64_t loc_or = 0, loc_and_inv = 0;
  {
    unsigned long long less_r = (unsigned long long)(wbase & 0xFFFFFFFFll), eq_r = (unsigned long long)(wbase >> 32);
    for (int64_t g0 = w0; g0 < w1; g0 += kW * 32) {
      uint64_t xs[kW];
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        const int64_t i = g0 + u * 32 + lane;
        xs[u] = i < w1 ? key_at(i) : kInf;
      }
#pragma unroll
      for (int u = 0; u < kW; ++u) {
        const int64_t i0 = g0 + u * 32;
        if (i0 >= w1) break;
        bool l, e;
        const uint64_t x = xs[u];
        classify_x(x, l, e);
        const unsigned bl = __ballot_sync(0xffffffffu, l), be = __ballot_sync(0xffffffffu, e);
        const unsigned long long lr = less_r + __popc(bl & lt), er = eq_r + __popc(be & lt);
        if (l || (e && er < quota)) {
          const unsigned long long pos = sel_before + lr + std::min(er, quota);
          pk0[pos] = x;
          pi0[pos] = (int32_t)(lo + i0 + lane);
          loc_or |= x;
          loc_and_inv |= ~x;
        }
        less_r += __popc(bl);
        eq_r += __popc(be);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    loc_or |= __shfl_xor_sync(0xffffffffu, loc_or, o);
    loc_and_inv |= __shfl_xor_sync(0xffffffffu, loc_and_inv, o);
  }
  if (lane == 0 && (loc_or | loc_and_inv)) {
    atomicOr(&sw->key_or, (unsigned long long)loc_or);
    atomicOr(&sw->key_and_inv, (unsigned long long)loc_and_inv);
  }
  if (c == 0 && tid == 0) *d_count = (int64_t)n_sel;
  stamp();
  grid.sync();
  const uint64_t vary = sw->key_or & sw->key_and_inv;  // bits that differ among selected keys

  stamp();
  // ---------------- 3. stable LSD radix sort of (key, id) by key ----------------
  // Only the bytes that vary among the selected keys are passes.  S sorter CTAs own contiguous
  // ranges of the array (<= one element per thread at k = 64k), cached in shared memory.
  // Per pass: digit bases = digits below (all sorters) + same digit in earlier sorters, read
  // from the [digit][sorter] count table; stable scatter chunk by chunk (warp match_any ranks
  // + exclusive per-warp digit prefix); the scatter also counts the NEXT pass's digits per
  // destination sorter, so each pass costs one grid barrier.  The last pass scatters ids
  // straight into out_ids.
  const int64_t m = (int64_t)n_sel;
  if (m == 0) return;
  int shifts[8], npass = 0;
#pragma unroll
  for (int b = 0; b < 8; ++b)
    if ((vary >> (8 * b)) & 0xFF) shifts[npass++] = 8 * b;
  if (npass == 0) {  // all selected keys equal: block-id order is the answer
    for (int64_t i = (int64_t)c * kThreads + tid; i < m; i += (int64_t)C * kThreads) out_ids[i] = pi0[i];
    return;
  }
  const int S = (int)std::min<int64_t>(C, (m + kThreads - 1) / kThreads);
  const int sper = (int)((m + S - 1) / S);
  const bool sorter = c < S;
  const int slo = sorter ? (int)std::min<int64_t>(m, (int64_t)c * sper) : 0;
  const int ns = sorter ? (int)std::min<int64_t>(m - slo, sper) : 0;
  const bool scache = cache_keys && (int64_t)ns * 12 <= per * 8;
  uint64_t *ck = s_keys;
  int32_t *ci = reinterpret_cast<int32_t *>(s_keys + ns);
  unsigned int *B[3] = {so->hist[0], so->hist[1], so->hist[2]};
  const int tbl = 256 * S;
  if (npass > 1)
    for (int e = c * kThreads + tid; e < tbl; e += C * kThreads) B[1][e] = 0u;
  uint64_t *ka = pk0, *kb = pk1;
  int32_t *ia = pi0, *ib = pi1;
  if (sorter) {  // pass-0 digit counts of this sorter's range
    for (int i = tid; i < 256; i += kThreads) s_hist[i] = 0;
    __syncthreads();
    for (int base = 0; base < ns; base += kThreads) {
      const int i = base + tid;
      uint64_t x = 0;
      if (i < ns) {
        x = ka[slo + i];
        if (scache) {
          ck[i] = x;
          ci[i] = ia[slo + i];
        }
      }
      hist_add_fast(s_hist, i < ns ? (int)((x >> shifts[0]) & 0xFF) : 256);
    }
    __syncthreads();
    for (int d = tid; d < 256; d += kThreads) B[0][c * 256 + d] = s_hist[d];
  }
  stamp();
  grid.sync();
  for (int pass = 0; pass < npass; ++pass) {
    const int shift = shifts[pass];
    const bool last = pass + 1 == npass;
    const int nshift = last ? 0 : shifts[pass + 1];
    unsigned int *Bc = B[pass % 3], *Bn = B[(pass + 1) % 3];
    if (pass + 2 < npass) {
      unsigned int *Bz = B[(pass + 2) % 3];
      for (int e = c * kThreads + tid; e < tbl; e += C * kThreads) Bz[e] = 0u;
    }
    if (sorter) {
      if (pass > 0 && scache) {
        for (int i = tid; i < ns; i += kThreads) {
          ck[i] = ka[slo + i];
          ci[i] = ia[slo + i];
        }
      }
      {  // digit bases: two threads per digit, each summing half of the sorter rows
        const int d = tid & 255, half = tid >> 8;
        const int hS = (S + 1) >> 1;
        const int ja = half * hS, jb = min(S, ja + hS);
        unsigned int tot = 0, earlier = 0;
        // latency-bound (L2 round trips): every load of a batch is issued before any is used
        constexpr int kBatch = 40;
        for (int j0 = ja; j0 < jb; j0 += kBatch) {
          unsigned int v[kBatch];
#pragma unroll
          for (int q = 0; q < kBatch; ++q) v[q] = j0 + q < jb ? __ldcg(Bc + (j0 + q) * 256 + d) : 0u;
#pragma unroll
          for (int q = 0; q < kBatch; ++q) {
            tot += v[q];
            earlier += j0 + q < c ? v[q] : 0u;
          }
        }
        if (half == 1) {
          s_part[d] = tot;
          s_base[d] = earlier;
        }
        __syncthreads();
        if (half == 0) {
          tot += s_part[d];
          earlier += s_base[d];
        }
        int all;
        const int below = block_excl_scan(half == 0 ? (int)tot : 0, s_warp, all);
        if (half == 0) s_base[d] = (unsigned int)below + earlier;
        __syncthreads();
      }
      stamp();
      for (int base = 0; base < ns; base += kThreads) {
        const int i = base + tid;
        const bool have = i < ns;
        const uint64_t x = have ? (scache ? ck[i] : ka[slo + i]) : 0;
        const int32_t xid = have ? (scache ? ci[i] : ia[slo + i]) : 0;
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
#pragma unroll
          for (int ww = 0; ww < kWarps; ++ww) {
            const unsigned int v = s_wcnt[ww][d];
            s_wcnt[ww][d] = acc;
            acc += v;
          }
        }
        __syncthreads();
        const unsigned int pos = have ? s_base[dg] + s_wcnt[w][dg] + wr : 0u;
        if (have) {
          if (last) {
            out_ids[pos] = xid;
          } else {
            kb[pos] = x;
            ib[pos] = xid;
          }
        }
        if (!last) {  // next pass's digit counts per destination sorter (warp-aggregated)
          const int nd = (int)((x >> nshift) & 0xFF);
          const int key2 = have ? (int)(pos / (unsigned)sper) * 256 + nd : -1;
          const unsigned p2 = __match_any_sync(0xffffffffu, key2);
          if (have && __popc(p2 & lanemask_lt()) == 0)
            atomicAdd(&Bn[key2], (unsigned)__popc(p2));  // [dest sorter][digit]
        }
        __syncthreads();
        if (have && wr == 0) atomicAdd(&s_base[dg], (unsigned)__popc(peers));  // next chunk
        __syncthreads();
      }
    }
    stamp();
    if (!last) {
      grid.sync();
      stamp();
      uint64_t *tk = ka; ka = kb; kb = tk;
      int32_t *ti = ia; ia = ib; ib = ti;
    }
  }
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
  const int nsm = sm_count();
  static int max_smem = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
  }();
  // half the SMs: the selection is latency-bound, and runs concurrently with the attention
  // kernels (whose CTAs take the other SMs / share these)
  int C = std::max(1, std::min(nsm / 2, kMaxCtas));
  if (const char *e = getenv("KVA_EVICT_CTAS")) C = std::max(1, std::min(atoi(e), std::min(nsm, kMaxCtas)));
  const int64_t per = (((n + C - 1) / C) + 1) & ~1ll;  // as in the kernel
  const size_t static_smem = 3 * 256 * 4 + 32 * 4 + 2 * 32 * 8 + 4 * 8 + kWarps * 256 * 4 + 1024;
  size_t dyn = (size_t)per * sizeof(uint64_t);
  // Keys are re-read from L2 each round by default (8 MB << 126 MB L2): without the 110 KB
  // shared-memory slice cache a selection CTA co-resides with a decode CTA, which measured
  // better for the whole step although the kernel alone is ~15% slower.
  // KVA_EVICT_CACHE=1 caches the slice in shared memory.
  int cache = 0;
  if (const char *e = getenv("KVA_EVICT_CACHE")) cache = atoi(e) != 0;
  if (!cache || dyn + static_smem > (size_t)max_smem) { dyn = 0; cache = 0; }
  // max dynamic smem + full carveout (CTAs of concurrently running kernels share SMs), once
  cudaError_t e = smem_attrs_once(reinterpret_cast<const void *>(evict_select_kernel), (int)dyn);
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
  // fast path region after the cooperative kernel's scratch
  p = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255));
  FastWs *fw = reinterpret_cast<FastWs *>(p);
  p += (sizeof(FastWs) + 255) & ~size_t(255);
  uint64_t *bkey = reinterpret_cast<uint64_t *>(p);
  p += (size_t)kBuckets * kCap * 8;
  int32_t *bid = reinterpret_cast<int32_t *>(p);
  p += (size_t)kBuckets * kCap * 4;
  if ((size_t)(p - reinterpret_cast<uint8_t *>(ws)) > ws_bytes) return cudaErrorInvalidValue;
  // KVA_EVICT_IMPL=fast selects the sample-bucket path (read per call).  Default: the
  // cooperative kernel alone — measured faster inside the bench step (its CTAs are resident
  // from the start and co-run with the decode kernel; the fast path's 64 x 1024-thread sort
  // CTAs queue behind it: 151 us alone vs 123, step 517 vs 455 us, profiles/r01b).
  const char *impl_env = getenv("KVA_EVICT_IMPL");
  const bool fast = impl_env && std::string(impl_env) == "fast" && n >= (1 << 16);
  const int *run_flag = nullptr;
  if (fast) {
    sel_sample_kernel<<<1, 1024, 0, s>>>(keys, n, k, fw);
    sel_bucket_kernel<<<std::max(1, std::min(nsm * 4, (int)((n + 4095) / 4096))), 256, 0, s>>>(keys, n, fw, bkey, bid);
    static bool attr = (cudaFuncSetAttribute(sel_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             kCap * 12), true);
    (void)attr;
    sel_sort_kernel<<<kBuckets, 1024, kCap * 12, s>>>(k, fw, bkey, bid, out_ids, d_count);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    run_flag = &fw->run_fallback;
  }
  e = cudaMemsetAsync(sw, 0, sizeof(SelWs), s);
  if (e != cudaSuccess) return e;
  void *args[] = {(void *)&keys, (void *)&n, (void *)&k, (void *)&out_ids, (void *)&d_count,
                  (void *)&sw, (void *)&so, (void *)&pk0, (void *)&pi0, (void *)&pk1, (void *)&pi1,
                  (void *)&cache, (void *)&run_flag};
  return cudaLaunchCooperativeKernel((void *)evict_select_kernel, dim3(C), dim3(kThreads), args, dyn, s);
}

}  // namespace kva
