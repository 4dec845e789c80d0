// kernels_evict.cu — task-aware eviction: priority keys and the radix
// top-k that replaces the paper's host-side free-table priority queue.
//
// Order: "When evicting the KV cache, we will first consider the priority of the KV cache
// entry, and then the last access time"; priorities P:331-334.  Keys are
// order-preserving u64 codes (readings #18-#20); equal keys are broken by block id.
//
// The selection itself (evict_select) is in kernels_select.cu.
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
constexpr int kMgrIndCap = 2048;  // chain-index entries kept in shared memory (8 KB: leaves room for 2 decode CTAs)

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
// KV-manager step: one cooperative kernel, phases separated by grid barriers.
// Transitions arrive as the caller's raw chains (host validated, uploaded unchanged); "last
// chain wins" is resolved on the device: every listed block's winner slot is reset, then
// takes the max element index listing it (atomicMax), and only that element applies its
// chain's state.  Then the reference counts (recount: zeroed + atomicAdd; incremental:
// atomicAdd / atomicSub), then keys + active count.
//   phase 0  rc = 0 (recount), win[id] = -1 for listed ids, *n_active = 0
//   phase 1  win[id] = max element index listing id
//   phase 2  winners apply (state, lat = now); rc += pool chains, -= deleted chains
//   phase 3  keys (evict_keys' encoding) + active count
__global__ void __launch_bounds__(256) manager_kernel(const __grid_constant__ MgrArgs a) {
  cg::grid_group grid = cg::this_grid();
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  if (a.span && t0 == 0) a.span[0] = gtime();
  __shared__ int32_t s_ind[kMgrIndCap];
  manager_phases(a, t0, nt, [&] { grid.sync(); }, s_ind, kMgrIndCap);
  // phase 3: 4 blocks per thread with vector loads/stores when the arrays allow it (torch
  // allocations are 256-B aligned), scalar tail
  unsigned act = 0;
  const uint8_t *state = a.state;
  const uint32_t *rc = a.rc, *lat = a.lat;
  const uint16_t *depth = a.depth;
  uint64_t *keys = a.keys;
  const bool vec = ((reinterpret_cast<uintptr_t>(state) | reinterpret_cast<uintptr_t>(rc) |
                     reinterpret_cast<uintptr_t>(lat) | reinterpret_cast<uintptr_t>(keys) |
                     (depth ? reinterpret_cast<uintptr_t>(depth) : 0)) & 15) == 0;
  const int64_t n4 = vec ? a.n / 4 : 0;
  for (int64_t q = t0; q < n4; q += nt) {
    const uint32_t s4 = __ldcg(reinterpret_cast<const uint32_t *>(state) + q);
    const uint4 r4 = __ldcg(reinterpret_cast<const uint4 *>(rc) + q);
    const uint4 l4 = __ldcg(reinterpret_cast<const uint4 *>(lat) + q);
    uint2 d4 = make_uint2(0u, 0u);
    if (depth) d4 = reinterpret_cast<const uint2 *>(depth)[q];
    const uint64_t k0 = manager_key(s4 & 0xFF, r4.x, l4.x, d4.x & 0xFFFF, act);
    const uint64_t k1 = manager_key((s4 >> 8) & 0xFF, r4.y, l4.y, d4.x >> 16, act);
    const uint64_t k2 = manager_key((s4 >> 16) & 0xFF, r4.z, l4.z, d4.y & 0xFFFF, act);
    const uint64_t k3 = manager_key(s4 >> 24, r4.w, l4.w, d4.y >> 16, act);
    reinterpret_cast<ulonglong2 *>(keys)[2 * q] = make_ulonglong2(k0, k1);
    reinterpret_cast<ulonglong2 *>(keys)[2 * q + 1] = make_ulonglong2(k2, k3);
  }
  for (int64_t b = 4 * n4 + t0; b < a.n; b += nt)
    keys[b] = manager_key(__ldcg(state + b), __ldcg(rc + b), __ldcg(lat + b), depth ? depth[b] : 0u, act);
  if (a.n_active) {  // one atomic per CTA (a per-warp atomic on one address serialises in L2)
    __shared__ unsigned int s_act;
    if (threadIdx.x == 0) s_act = 0u;
    __syncthreads();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) act += __shfl_xor_sync(0xffffffffu, act, o);
    if ((threadIdx.x & 31) == 0 && act) atomicAdd(&s_act, act);
    __syncthreads();
    if (threadIdx.x == 0 && s_act) atomicAdd(a.n_active, (unsigned long long)s_act);
  }
  if (a.span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.span + 1, gtime());
  }
}

cudaError_t launch_manager_step(uint8_t *state, uint32_t *rc, uint32_t *lat, const uint16_t *depth,
                                int64_t n, uint32_t now, const int32_t *tr_ids, int64_t n_tr,
                                const int32_t *tr_indptr, const uint8_t *tr_state, int32_t n_chains,
                                int32_t *win, bool recount, const int32_t *pool_ids, int64_t pool_len,
                                const int32_t *del_ids, int64_t del_len, uint64_t *keys, int64_t *n_active,
                                cudaStream_t s) {
  MgrArgs a = make_mgr_args(state, rc, lat, depth, n, now, tr_ids, n_tr, tr_indptr, tr_state, n_chains, win,
                            recount, pool_ids, pool_len, del_ids, del_len, keys, n_active);
  a.span = span_ring_slot(0);
  if (n <= 0 && n_active == nullptr) return cudaSuccess;
  // two 256-thread CTAs per SM (co-resident on an idle GPU: cooperative launch); every phase is
  // a grid-stride pass over <= 2^20 elements (a few per thread)
  const int grid = std::max(1, std::min<int>(2 * sm_count(), (int)((std::max<int64_t>(n, n_tr + pool_len + del_len) + 255) / 256)));
  void *args[] = {(void *)&a};
  return cudaLaunchCooperativeKernel((void *)manager_kernel, dim3(grid), dim3(256), args, 0, s);
}

// Release: set the free bits of the listed blocks and (truncate) write -1 into the listed
// block-table entries.  The lists travel as a kernel parameter (no upload); capacity templated
// so that a short list does not pay for a 30 KB parameter block.
template <int CAP>
struct ReleaseList {
  int32_t n;
  int32_t *table;  // nullable: entries tbl[0, n) are set to -1
  int32_t ids[CAP];
  int32_t tbl[CAP];
};
template <int CAP>
__global__ void release_ids_kernel(uint32_t *free_bits, const __grid_constant__ ReleaseList<CAP> r,
                                   unsigned long long *span) {
  // a programmatic dependent of the preceding kernel (option pdl): waits for it first
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (span && blockIdx.x == 0 && threadIdx.x == 0) span[0] = gtime();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r.n; i += gridDim.x * blockDim.x) {
    atomicOr(free_bits + (r.ids[i] >> 5), 1u << (r.ids[i] & 31));
    if (r.table) r.table[r.tbl[i]] = -1;
  }
  if (span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(span + 1, gtime());
  }
}
template <int CAP>
static cudaError_t release_launch(uint32_t *free_bits, const int32_t *ids, const int32_t *tbl, int32_t *table, int n,
                                  cudaStream_t s) {
  ReleaseList<CAP> r;
  r.n = n;
  r.table = tbl ? table : nullptr;
  std::memcpy(r.ids, ids, sizeof(int32_t) * n);
  if (tbl) std::memcpy(r.tbl, tbl, sizeof(int32_t) * n);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = opt(kOptPdl) != 0 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, release_ids_kernel<CAP>, free_bits, r, span_ring_slot(4));
}

cudaError_t launch_release_ids(uint32_t *free_bits, const int32_t *ids_host, int n, cudaStream_t s,
                               const int32_t *tbl_host, int32_t *table) {
  if (n <= 0) return cudaSuccess;
  if (n <= 256) return release_launch<256>(free_bits, ids_host, tbl_host, table, n, s);
  return release_launch<kReleaseBatch>(free_bits, ids_host, tbl_host, table, n, s);
}

}  // namespace kva
