// kernels_merge_append.cu — LSE merge of partial softmax states and the
// coalesced KV-append block scatter (a2).
#include <math_constants.h>

#include "kvattn.h"
#include "common.cuh"
#include "internal.h"

namespace kva {
using namespace dev;

// ---------------------------------------------------------------------------------------
// a6: for each output (row, q-head) with partials {(O_j, lse_j)}:
//   lse = ln sum_j e^{lse_j},  O = sum_j e^{lse_j - lse} O_j.
// One warp per (request row, kv head); each lane owns D/32 contiguous channels (16-B / 8-B
// vectors).  Partials in order: the cascade prefix slots (one per nested level), then the key
// splits.
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256) merge_kernel(const AttnParams p,
                                                    const __grid_constant__ ReqList<MergeReq> RL,
                                                    int n_units) {
  constexpr int V = D / 32;  // 4 (d=128) or 2 (d=64)
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n_units) return;
  const int m = w / p.Hkv, h = w - m * p.Hkv;  // m = (request, row)
  const MergeReq *reqs = RL.ptr ? RL.ptr : RL.req;
  const int32_t *pre = RL.ptr ? RL.pre_ptr : RL.pre;
  int lo = 0, hi = RL.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pre[mid] <= m) lo = mid;
    else hi = mid - 1;
  }
  const MergeReq mq = reqs[lo];
  const int r = m - pre[lo];
  const int nc = mq.n_casc;
  const int n = nc + mq.nsplit;
  const int split0 = mq.split_slot + h * mq.nsplit * mq.rows + r;
  auto slot_of = [&](int i) {
    return i < nc ? mq.casc_slot[i] + h * mq.casc_hstride[i] + r : split0 + (i - nc) * mq.rows;
  };
  float L = -CUDART_INF_F;
  for (int i = lane; i < n; i += 32) L = fmaxf(L, p.part_lse[slot_of(i)]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) L = fmaxf(L, __shfl_xor_sync(0xffffffffu, L, o));
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float sum = 0.f;
  for (int i = 0; i < n; ++i) {
    const int sl = slot_of(i);
    const float lj = __ldg(p.part_lse + sl);
    const float wgt = lj == -CUDART_INF_F ? 0.f : __expf(lj - L);
    sum += wgt;
    const float *src = p.part_o + (int64_t)sl * D + lane * V;
    if constexpr (V == 4) {
      const float4 x = __ldg(reinterpret_cast<const float4 *>(src));
      acc[0] += wgt * x.x; acc[1] += wgt * x.y; acc[2] += wgt * x.z; acc[3] += wgt * x.w;
    } else {
      const float2 x = __ldg(reinterpret_cast<const float2 *>(src));
      acc[0] += wgt * x.x; acc[1] += wgt * x.y;
    }
  }
  const float inv = 1.f / sum;
  const int q_head = h * p.g + r % p.g, q_row = mq.q_row0 + r / p.g;
  const int64_t off = (int64_t)q_row * p.o_stride_tok + (int64_t)q_head * p.o_stride_head + lane * V;
  if (p.out_f32) {
    float *dst = reinterpret_cast<float *>(p.out) + off;
    if constexpr (V == 4)
      *reinterpret_cast<float4 *>(dst) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
    else
      *reinterpret_cast<float2 *>(dst) = make_float2(acc[0] * inv, acc[1] * inv);
  } else {
    uint16_t *dst = reinterpret_cast<uint16_t *>(p.out) + off;
    if constexpr (V == 4)
      *reinterpret_cast<uint2 *>(dst) = make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv),
                                                   pack_bf16(acc[2] * inv, acc[3] * inv));
    else
      *reinterpret_cast<uint32_t *>(dst) = pack_bf16(acc[0] * inv, acc[1] * inv);
  }
  if (p.lse && lane == 0) p.lse[(int64_t)q_row * p.Hq + q_head] = L + __logf(sum);
}

cudaError_t launch_merge(const AttnParams &p, const ReqList<MergeReq> &RL, int n_units, cudaStream_t s) {
  if (n_units <= 0) return cudaSuccess;
  const int grid = (n_units + 7) / 8;
  if (p.d == 128)
    merge_kernel<128><<<grid, 256, 0, s>>>(p, RL, n_units);
  else
    merge_kernel<64><<<grid, 256, 0, s>>>(p, RL, n_units);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// a2: KV append.  (1) alloc_write publishes the ids the host allocator chose (smallest free
// first, reading #13) in the device block table and clears their free bits; (2) the scatter
// copies every (new token, local kv-head) row of a request list (exclusive token prefix
// tok_pre) to slot (table[i][t/16], t % 16).
// ---------------------------------------------------------------------------------------
__global__ void alloc_write_kernel(int32_t *__restrict__ block_table, uint32_t *__restrict__ free_bits,
                                   const __grid_constant__ AllocList al) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= al.n) return;
  const int32_t id = al.ids_ptr ? al.ids_ptr[i] : al.ids[i];
  block_table[al.tbl_ptr ? al.tbl_ptr[i] : al.tbl[i]] = id;
  atomicAnd(free_bits + (id >> 5), ~(1u << (id & 31)));
}

cudaError_t launch_alloc_write(int32_t *block_table, uint32_t *free_bits, const AllocList &al, cudaStream_t s) {
  if (al.n <= 0) return cudaSuccess;
  alloc_write_kernel<<<(al.n + 255) / 256, 256, 0, s>>>(block_table, free_bits, al);
  return cudaGetLastError();
}

// One CTA moves kUnitsPerCta (token, kv-head) rows of K and V: phase 1 resolves each unit's
// destination slot (binary search of q_indptr + one table read) into shared memory, phase 2
// copies with every thread issuing all its 16-byte loads before its stores (ILP).
constexpr int kUnitsPerCta = 32;
__global__ void __launch_bounds__(256) append_kernel(
    const uint16_t *__restrict__ k_new, const uint16_t *__restrict__ v_new, int64_t stride_tok,
    uint16_t *__restrict__ k_pool, uint16_t *__restrict__ v_pool, int32_t Hkv, int32_t d,
    const int32_t *__restrict__ block_table, int32_t max_blocks, const __grid_constant__ ReqList<AppendReq> L,
    int32_t total_new_tok, int32_t early_trigger) {
  // early_trigger (the append of the tile-path rows only): the tile kernel launched right
  // after it (programmatic dependent launch) may become resident now; it waits
  // (griddepcontrol.wait) before reading the pool.  The decode kernel, a dependent of the tile
  // kernel that does NOT wait, reads only decode-class rows, which an earlier append on the
  // stream wrote.  The decode-class append never triggers early: a tile kernel launched right
  // after it (no tile-path rows) starts only once those rows are complete, and so does the
  // decode kernel behind it.
  if (early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const AppendReq *reqs = L.ptr ? L.ptr : L.req;
  const int32_t *tok_pre = L.ptr ? L.pre_ptr : L.pre;
  const int num_reqs = L.n;
  __shared__ int64_t s_src[kUnitsPerCta], s_dst[kUnitsPerCta];
  const int64_t n_units = (int64_t)total_new_tok * Hkv;
  const int64_t u0 = (int64_t)blockIdx.x * kUnitsPerCta;
  if (threadIdx.x < kUnitsPerCta) {
    const int64_t unit = u0 + threadIdx.x;
    int64_t src = -1, dst = -1;
    if (unit < n_units) {
      const int j = (int)(unit / Hkv), h = (int)(unit % Hkv);  // j-th new token of the list
      int lo = 0, hi = num_reqs - 1;  // its request: last i with tok_pre[i] <= j
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (tok_pre[mid] <= j) lo = mid; else hi = mid - 1;
      }
      const AppendReq rq = reqs[lo];
      const int off = j - tok_pre[lo];
      const int t = rq.pos0 + off;
      const int32_t id = block_table[(int64_t)rq.table_row * max_blocks + t / kBlock];
      src = (int64_t)(rq.q_row0 + off) * stride_tok + (int64_t)h * d;
      dst = (((int64_t)id * Hkv + h) * kBlock + t % kBlock) * d;
    }
    s_src[threadIdx.x] = src;
    s_dst[threadIdx.x] = dst;
  }
  __syncthreads();
  const int cpr = d / 8;                    // 16-byte chunks per row
  const int per_unit = 2 * cpr;             // K and V
  const int total = kUnitsPerCta * per_unit;
  constexpr int kMaxIt = kUnitsPerCta * 2 * 16 / 256;  // 4 for d = 128
  uint4 v[kMaxIt];
  int64_t dsto[kMaxIt];
  bool isv[kMaxIt];
#pragma unroll
  for (int k = 0; k < kMaxIt; ++k) {
    const int c = threadIdx.x + k * 256;
    dsto[k] = -1;
    if (c < total) {
      const int u = c / per_unit, r = c % per_unit;
      const int tensor = r / cpr, part = r % cpr;
      if (s_src[u] >= 0) {
        isv[k] = tensor;
        v[k] = __ldg(reinterpret_cast<const uint4 *>((tensor ? v_new : k_new) + s_src[u] + part * 8));
        dsto[k] = s_dst[u] + part * 8;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxIt; ++k)
    if (dsto[k] >= 0) *reinterpret_cast<uint4 *>((isv[k] ? v_pool : k_pool) + dsto[k]) = v[k];
}

cudaError_t launch_append(const uint16_t *k_new, const uint16_t *v_new, int64_t stride_tok,
                          uint16_t *k_pool, uint16_t *v_pool, int32_t Hkv, int32_t d,
                          const int32_t *block_table, int32_t max_blocks,
                          const ReqList<AppendReq> &L, int32_t total_new_tok, cudaStream_t s,
                          bool early_trigger) {
  const int64_t units = (int64_t)total_new_tok * Hkv;
  if (units <= 0 || L.n <= 0) return cudaSuccess;
  static bool carve = (cudaFuncSetAttribute(append_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared), true);
  (void)carve;
  append_kernel<<<(unsigned)((units + kUnitsPerCta - 1) / kUnitsPerCta), 256, 0, s>>>(
      k_new, v_new, stride_tok, k_pool, v_pool, Hkv, d, block_table, max_blocks, L, total_new_tok,
      early_trigger ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace kva

// ------------------------------------------------------------------------------------------
// Diagnostics only (kva_diag_occupy): n_ctas CTAs that each hold `smem` bytes of shared
// memory and spin for `ns` nanoseconds, so a kernel launched next on another stream runs on
// the remaining SMs (measures a kernel's throughput as a function of the SMs it gets).
namespace kva {
__global__ void diag_occupy_kernel(unsigned long long ns) {
  extern __shared__ uint8_t sm_pad[];
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  if (threadIdx.x == 0) sm_pad[0] = 0;
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
}  // namespace kva

extern "C" kva_status kva_diag_occupy(int32_t n_ctas, int32_t smem_bytes, int64_t ns, kva_stream_t stream) {
  if (n_ctas <= 0) return KVA_OK;
  if (cudaFuncSetAttribute(kva::diag_occupy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess)
    return KVA_ERR_CUDA;
  kva::diag_occupy_kernel<<<n_ctas, 32, smem_bytes, reinterpret_cast<cudaStream_t>(stream)>>>((unsigned long long)ns);
  return cudaGetLastError() == cudaSuccess ? KVA_OK : KVA_ERR_CUDA;
}
