// kernels_evict.cu — task-aware eviction: priority keys and the radix
// top-k that replaces the paper's host-side free-table priority queue.
//
// Order: "When evicting the KV cache, we will first consider the priority of the KV cache
// entry, and then the last access time"; priorities P:331-334.  Keys are
// order-preserving u64 codes (readings #18-#20); equal keys are broken by block id.
//
// The selection itself (evict_select) is in kernels_select.cu.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

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

}  // namespace kva
