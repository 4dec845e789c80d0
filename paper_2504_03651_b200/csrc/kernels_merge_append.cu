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
// One HALF-warp per (request row, kv head) — two units per warp instruction stream, each lane
// owning D/16 contiguous channels (2 x 16-B for d = 128).  Partials in order: the cascade
// prefix slots (one per nested level), then the key splits.  lse and O of up to kBatch
// partials are loaded in one memory round trip, before the max (which they do not need).
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(256, 4) merge_kernel(const AttnParams p,
                                                    const __grid_constant__ ReqList<MergeReq> RL,
                                                    int n_units) {
  constexpr int V = D / 16;  // channels per lane: 8 (d=128) or 4 (d=64)
  constexpr int kUnitsPerCta = 16;
  const int lane = threadIdx.x & 31, hl = lane & 15;  // lane within the half-warp
  const unsigned hmask = (lane < 16) ? 0x0000FFFFu : 0xFFFF0000u;
  const int w = blockIdx.x * kUnitsPerCta + (threadIdx.x >> 4);  // this half-warp's unit
  // the next launch on the stream (kv_truncate's release, the next kv_append: programmatic
  // dependents that wait for this grid before touching memory) may be set up now
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.span && threadIdx.x == 0) {  // instrumentation: CTA start
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    atomicMin(&p.span[4], t0);
  }
  const MergeReq *reqs = RL.ptr ? RL.ptr : RL.req;
  const int32_t *pre = RL.ptr ? RL.pre_ptr : RL.pre;
  // the request of the CTA's first unit by one binary search (warp 0), shared; each half-warp
  // walks forward from it (its unit is at most 15 further: usually the same request)
  __shared__ int s_req0;
  __shared__ unsigned s_fin;
  if (threadIdx.x == 0) s_fin = 0u;
  if (threadIdx.x < 32) {
    const int m0 = min(blockIdx.x * kUnitsPerCta, n_units - 1) / p.Hkv;
    int lo = 0, hi = RL.n - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pre[mid] <= m0) lo = mid;
      else hi = mid - 1;
    }
    if (threadIdx.x == 0) s_req0 = lo;
  }
  __syncthreads();
  if (w >= n_units) return;  // whole half-warps leave (n_units is a per-half-warp bound)
  const int m = w / p.Hkv, h = w - m * p.Hkv;  // m = (request, row)
  int lo = s_req0;
  while (lo + 1 < RL.n && pre[lo + 1] <= m) ++lo;
  const MergeReq &mq = reqs[lo];  // (a reference: dynamic casc_slot[i] indexing without a stack copy)
  const int r = m - pre[lo];
  const int nc = mq.n_casc;
  const int n = nc + mq.nsplit;
  const int split0 = mq.split_slot + h * mq.nsplit * mq.rows + r;
  auto slot_of = [&](int i) {
    return i < nc ? mq.casc_slot[i] + h * mq.casc_hstride[i] + r : split0 + (i - nc) * mq.rows;
  };
  constexpr int kBatch = 4;
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  float sum = 0.f, L = -CUDART_INF_F;
  for (int i0 = 0; i0 < n; i0 += kBatch) {  // (the two half-warps may run different counts)
    const int nb = min(kBatch, n - i0);
    const float lj = hl < nb ? __ldg(p.part_lse + slot_of(i0 + hl)) : -CUDART_INF_F;
    float xs[kBatch][V];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      if (j < nb) {
        const float4 *src = reinterpret_cast<const float4 *>(p.part_o + (int64_t)slot_of(i0 + j) * D + hl * V);
#pragma unroll
        for (int v4 = 0; v4 < V / 4; ++v4) {
          const float4 x = __ldg(src + v4);
          xs[j][4 * v4] = x.x; xs[j][4 * v4 + 1] = x.y; xs[j][4 * v4 + 2] = x.z; xs[j][4 * v4 + 3] = x.w;
        }
      }
    }
    float bm = lj;
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) bm = fmaxf(bm, __shfl_xor_sync(hmask, bm, o, 16));
    const float Ln = fmaxf(L, bm);
    if (Ln != L && L != -CUDART_INF_F) {  // a later batch raised the max (n > kBatch only)
      const float c = __expf(L - Ln);
      sum *= c;
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] *= c;
    }
    L = Ln;
    const float my_w = lj == -CUDART_INF_F ? 0.f : __expf(lj - L);
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const float wgt = __shfl_sync(hmask, my_w, j, 16);
      if (j < nb) {
        sum += wgt;
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] += wgt * xs[j][v];
      }
    }
  }
  const float inv = 1.f / sum;
  const int q_head = h * p.g + r % p.g, q_row = mq.q_row0 + r / p.g;
  const int64_t off = (int64_t)q_row * p.o_stride_tok + (int64_t)q_head * p.o_stride_head + hl * V;
  for (int o = 0; o <= p.n_out_extra; ++o) {  // own output, then the peers' (fused a7)
    void *base = o == 0 ? p.out : p.out_extra[o - 1];
    if (p.out_f32) {
      float4 *dst = reinterpret_cast<float4 *>(reinterpret_cast<float *>(base) + off);
#pragma unroll
      for (int v4 = 0; v4 < V / 4; ++v4)
        dst[v4] = make_float4(acc[4 * v4] * inv, acc[4 * v4 + 1] * inv, acc[4 * v4 + 2] * inv, acc[4 * v4 + 3] * inv);
    } else {
      uint16_t *dst = reinterpret_cast<uint16_t *>(base) + off;
      if constexpr (V == 8) {
        *reinterpret_cast<uint4 *>(dst) = make_uint4(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv),
                                                     pack_bf16(acc[4] * inv, acc[5] * inv), pack_bf16(acc[6] * inv, acc[7] * inv));
      } else {
        *reinterpret_cast<uint2 *>(dst) = make_uint2(pack_bf16(acc[0] * inv, acc[1] * inv), pack_bf16(acc[2] * inv, acc[3] * inv));
      }
    }
  }
  if (p.lse && hl == 0) p.lse[(int64_t)q_row * p.Hq + q_head] = L + __logf(sum);
  if (p.span) {  // instrumentation: the CTA's last unit to finish records the end
    if (hl == 0) {
      const unsigned active = min(kUnitsPerCta, n_units - (int)blockIdx.x * kUnitsPerCta);
      if (atomicAdd(&s_fin, 1u) + 1 == active) {
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        atomicMax(&p.span[5], t1);
      }
    }
  }
}

__global__ void join_kernel() {}
cudaError_t launch_join(cudaStream_t s) {
  join_kernel<<<1, 32, 0, s>>>();
  return cudaGetLastError();
}

cudaError_t launch_merge(const AttnParams &p, const ReqList<MergeReq> &RL, int n_units, cudaStream_t s) {
  if (n_units <= 0) return cudaSuccess;
  const int grid = (n_units + 15) / 16;  // 16 units (half-warps) per 256-thread CTA
  if (p.d == 128)
    merge_kernel<128><<<grid, 256, 0, s>>>(p, RL, n_units);
  else
    merge_kernel<64><<<grid, 256, 0, s>>>(p, RL, n_units);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------
// a2: KV append.  The scatter copies every (new token, local kv-head) row of a request list
// (exclusive token prefix tok_pre) to slot (block(t/16), t % 16), the block id taken from the
// request's host-resolved ids (decode-class) or the block table.  The launch of the
// decode-class list also publishes the ids the host allocator chose (smallest free first,
// reading #13): table entries written and free bits cleared by its trailing CTAs.
// ---------------------------------------------------------------------------------------
// One CTA moves kUnitsPerCta (token, kv-head) rows of K and V: phase 1 resolves each unit's
// destination slot (binary search of q_indptr + the request's block id) into shared memory,
// phase 2 copies with every thread issuing all its 16-byte loads before its stores (ILP).
constexpr int kUnitsPerCta = 32;
struct AppendArgs {
  const uint16_t *k_new, *v_new;
  int64_t stride_tok;
  uint16_t *k_pool, *v_pool;
  int32_t Hkv, d;
  int32_t *block_table;
  int32_t max_blocks, total_new_tok, early_trigger, n_app_ctas;
  uint32_t *free_bits;
  unsigned long long *span;  // diagnostics (span_ring)
};
template <bool ALLOC>
struct AllocParam {
  AllocList al;
};
template <>
struct AllocParam<false> {};

template <bool ALLOC>
__global__ void __launch_bounds__(256) append_kernel(const __grid_constant__ AppendArgs a,
                                                     const __grid_constant__ ReqList<AppendReq> L,
                                                     const __grid_constant__ AllocParam<ALLOC> ap) {
  // early_trigger, after the wait: the append of the tile-path rows — the tile kernel launched
  // right after it (programmatic dependent launch) may become resident now; it waits
  // (griddepcontrol.wait) before reading the pool.  The decode kernel, a dependent of the tile
  // kernel that does NOT wait, reads only decode-class rows, which the preceding append wrote
  // (complete: this kernel waited for it).  The decode-class append triggers early only when
  // the tile-path append follows it (that one waits); with no tile-path rows the tile kernel
  // follows it directly and starts only once it is complete, and so does the decode kernel.
  // launched as a programmatic dependent of the preceding kernel (option pdl): its setup
  // overlaps that kernel, and nothing is read or written before it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.span && blockIdx.x == 0 && threadIdx.x == 0) a.span[0] = gtime();
  if constexpr (ALLOC) {
    if ((int)blockIdx.x >= a.n_app_ctas) {  // allocation publishing
      const AllocList &al = ap.al;
      const int i = ((int)blockIdx.x - a.n_app_ctas) * blockDim.x + threadIdx.x;
      if (i >= al.n) return;
      const int32_t id = al.ids_ptr ? al.ids_ptr[i] : al.ids[i];
      a.block_table[al.tbl_ptr ? al.tbl_ptr[i] : al.tbl[i]] = id;
      atomicAnd(a.free_bits + (id >> 5), ~(1u << (id & 31)));
      return;
    }
  }
  const AppendReq *reqs = L.ptr ? L.ptr : L.req;
  const int32_t *tok_pre = L.ptr ? L.pre_ptr : L.pre;
  const int num_reqs = L.n;
  const int Hkv = a.Hkv, d = a.d;
  __shared__ int64_t s_src[kUnitsPerCta], s_dst[kUnitsPerCta];
  const int64_t n_units = (int64_t)a.total_new_tok * Hkv;
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
      const int32_t id = rq.blk[0] >= 0 ? rq.blk[t / kBlock - rq.pos0 / kBlock]
                                        : a.block_table[(int64_t)rq.table_row * a.max_blocks + t / kBlock];
      src = (int64_t)(rq.q_row0 + off) * a.stride_tok + (int64_t)h * d;
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
        v[k] = __ldg(reinterpret_cast<const uint4 *>((tensor ? a.v_new : a.k_new) + s_src[u] + part * 8));
        dsto[k] = s_dst[u] + part * 8;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxIt; ++k)
    if (dsto[k] >= 0) *reinterpret_cast<uint4 *>((isv[k] ? a.v_pool : a.k_pool) + dsto[k]) = v[k];
  if (a.span) {
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(a.span + 1, gtime());
  }
}

cudaError_t launch_append(const uint16_t *k_new, const uint16_t *v_new, int64_t stride_tok,
                          uint16_t *k_pool, uint16_t *v_pool, int32_t Hkv, int32_t d,
                          int32_t *block_table, int32_t max_blocks,
                          const ReqList<AppendReq> &L, int32_t total_new_tok, cudaStream_t s,
                          bool early_trigger, const AllocList *al, uint32_t *free_bits) {
  const int64_t units = L.n > 0 ? (int64_t)total_new_tok * Hkv : 0;
  const int n_app = (int)((units + kUnitsPerCta - 1) / kUnitsPerCta);
  const int n_alloc = al ? (al->n + 255) / 256 : 0;
  if (n_app + n_alloc <= 0) return cudaSuccess;
  AppendArgs a{k_new, v_new, stride_tok, k_pool, v_pool, Hkv, d, block_table, max_blocks,
               total_new_tok, early_trigger ? 1 : 0, n_app, free_bits, span_ring_slot(al ? 2 : 3)};
  // programmatic dependent launch (option pdl): the kernel waits for its predecessor at its
  // first instruction, so only the launch latency overlaps
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = opt(kOptPdl) != 0 ? 1 : 0;
  if (al && al->n > 0) {
    static bool carve = (cudaFuncSetAttribute(append_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                              cudaSharedmemCarveoutMaxShared), true);
    (void)carve;
    AllocParam<true> ap;
    ap.al = *al;
    cfg.gridDim = dim3((unsigned)(n_app + n_alloc));
    return cudaLaunchKernelEx(&cfg, append_kernel<true>, a, L, ap);
  }
  if (n_app <= 0) return cudaSuccess;
  static bool carve = (cudaFuncSetAttribute(append_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                            cudaSharedmemCarveoutMaxShared), true);
  (void)carve;
  cfg.gridDim = dim3((unsigned)n_app);
  return cudaLaunchKernelEx(&cfg, append_kernel<false>, a, L, AllocParam<false>{});
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
