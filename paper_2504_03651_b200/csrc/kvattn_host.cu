// kvattn_host.cu — the C ABI of include/kvattn.h: pool handle, host validation, the block
// allocator, the hybrid-attention planner, plan upload and launches.
// Product code; shares nothing with oracle/.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/kvattn.h"
#include "internal.h"

using namespace kva;

// ------------------------------------------------------------------------------------------
// host-side section timer (diagnostics): option "host_prof" = 1 accumulates steady-clock time
// per labelled section and prints the per-call medians / means at exit
// ------------------------------------------------------------------------------------------
namespace {
struct HostProf {
  std::mutex mu;
  std::vector<std::pair<std::string, std::vector<double>>> acc;
  void add(const char *name, double us) {
    std::lock_guard<std::mutex> g(mu);
    for (auto &a : acc)
      if (a.first == name) {
        a.second.push_back(us);
        return;
      }
    acc.push_back({name, {us}});
  }
  ~HostProf() {  // median and mean per label (first calls include lazy module loading)
    if (acc.empty()) return;
    for (auto &a : acc) {
      std::vector<double> v = a.second;
      std::sort(v.begin(), v.end());
      double m = 0;
      for (double x : v) m += x;
      fprintf(stderr, "[kva host] %-28s median %8.2f us  mean %8.2f us  (%zu calls)\n", a.first.c_str(),
              v[v.size() / 2], m / v.size(), v.size());
    }
  }
};
HostProf g_hprof;
struct HSection {  // HSection t; ... t.lap("label");
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void lap(const char *name) {
    if (!opt(kOptHostProf)) return;
    const auto n = std::chrono::steady_clock::now();
    g_hprof.add(name, std::chrono::duration<double, std::micro>(n - t).count());
    t = n;
  }
};
}  // namespace

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err = "";

static kva_status fail(kva_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess)                                                               \
      return fail(KVA_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, \
                  __LINE__);                                                             \
  } while (0)

extern "C" const char *kva_last_error(void) { return g_err.c_str(); }
namespace kva {
kva_status set_error(kva_status st, const char *msg) {
  g_err = msg;
  return st;
}
cudaError_t smem_attrs_once(const void *kern, int smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void *, int>, int>> done;  // ((kernel, device), smem)
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto &d : done)
      if (d.first.first == kern && d.first.second == dev && d.second >= smem) return cudaSuccess;
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lk(mu);
    done.push_back({{kern, dev}, smem});
  }
  return e;
}
int sm_count() {
  static int cached[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev]) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
}
namespace {
struct OptDef {
  const char *name;
  int64_t def;
};
// defaults = the measured best
constexpr OptDef kOptDefs[kOptCount] = {{"tile_ctas", 0}, {"overlap", 1}, {"pdl", 1},   {"evict_ctas", 0},
                                        {"host_prof", 0}, {"debug_flags", 0}, {"debug_ts", 0},
                                        {"span_ring", 0}, {"evict_threads", 512}, {"fold", 0}};
std::atomic<int64_t> g_opt[kOptCount] = {{0}, {1}, {1}, {0}, {0}, {0}, {0}, {0}, {512}, {0}};
std::atomic<unsigned> g_span_seq[5] = {{0}, {0}, {0}, {0}, {0}};
int opt_index(const char *name) {
  if (!name) return -1;
  for (int i = 0; i < kOptCount; ++i)
    if (std::strcmp(kOptDefs[i].name, name) == 0) return i;
  return -1;
}
}  // namespace
int64_t opt(Opt o) { return g_opt[o].load(std::memory_order_relaxed); }
size_t evict_select_ws_bytes(int64_t n, int64_t k) {
  return std::max(evict_select_ws_bytes_512(n, k), evict_select_ws_bytes_256(n, k));
}
cudaError_t launch_evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids, int64_t *d_count,
                                uint32_t *free_bits, void *ws, size_t ws_bytes, int ctas, cudaStream_t s,
                                const MgrArgs *mgr) {
  return opt(kOptEvictThreads) == 256
             ? launch_evict_select_256(keys, n, k, out_ids, d_count, free_bits, ws, ws_bytes, ctas, s, mgr)
             : launch_evict_select_512(keys, n, k, out_ids, d_count, free_bits, ws, ws_bytes, ctas, s, mgr);
}
unsigned long long *span_ring_slot(int kind) {
  const int64_t r = opt(kOptSpanRing);
  if (!r) return nullptr;
  const unsigned i = g_span_seq[kind].fetch_add(1u, std::memory_order_relaxed) & 255u;
  return reinterpret_cast<unsigned long long *>(r) + ((size_t)kind * 256 + i) * 2;
}
}  // namespace kva
extern "C" kva_status kva_set_option(const char *name, int64_t value) {
  const int i = kva::opt_index(name);
  if (i < 0) return fail(KVA_ERR_INVALID, "unknown option '%s'", name ? name : "(null)");
  if (i == kva::kOptEvictThreads && value != 256 && value != 512)
    return fail(KVA_ERR_INVALID, "evict_threads must be 256 or 512");
  kva::g_opt[i].store(value, std::memory_order_relaxed);
  return KVA_OK;
}
extern "C" kva_status kva_get_option(const char *name, int64_t *value) {
  const int i = kva::opt_index(name);
  if (i < 0 || !value) return fail(KVA_ERR_INVALID, "unknown option '%s' or null value", name ? name : "(null)");
  *value = kva::g_opt[i].load(std::memory_order_relaxed);
  return KVA_OK;
}
extern "C" const char *kva_version(void) {
  return "kvattn 0.1 (sm_100a; decode split-KV TMA+mma.sync, tile attention, radix top-k)";
}

namespace {

struct DeviceGuard {  // switch to the pool's device for the call, restore afterwards
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

// Pinned host staging ring for plan uploads (host -> workspace copies on the stream).
struct Staging {
  struct Slot {
    void *host = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  };
  Slot slot[4];
  int next = 0;
  cudaError_t get(size_t bytes, Slot **out) {
    Slot &s = slot[next];
    next = (next + 1) % 4;
    if (s.pending) {
      cudaError_t e = cudaEventSynchronize(s.ev);
      if (e != cudaSuccess) return e;
      s.pending = false;
    }
    if (!s.ev) {
      cudaError_t e = cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    if (s.cap < bytes) {
      if (s.host) cudaFreeHost(s.host);
      s.cap = std::max<size_t>(bytes, 1 << 16);
      cudaError_t e = cudaMallocHost(&s.host, s.cap);
      if (e != cudaSuccess) {
        s.host = nullptr;
        s.cap = 0;
        return e;
      }
    }
    *out = &s;
    return cudaSuccess;
  }
  cudaError_t upload(Slot *s, void *dev_dst, size_t bytes, cudaStream_t st) {
    cudaError_t e = cudaMemcpyAsync(dev_dst, s->host, bytes, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(s->ev, st);
    s->pending = (e == cudaSuccess);
    return e;
  }
  void release() {
    for (auto &s : slot) {
      if (s.pending) cudaEventSynchronize(s.ev);
      if (s.host) cudaFreeHost(s.host);
      if (s.ev) cudaEventDestroy(s.ev);
      s = Slot{};
    }
  }
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 2-D view of a pool tensor: dim0 = head_dim (contiguous), dim1 = num_blocks*Hkv*16 rows;
// box = 64 channels x 16 rows (one block-head half), 128-byte swizzle.
// 3-D view {64 channels, rows, 2 halves} of a d = 128 pool: ONE box {64, 16, 2} moves a whole
// block-head (4 KB) into shared memory as [half][16 rows][64] with the 128-B swizzle of each
// half — exactly the layout of two 2-D boxes, in half the TMA operations (the K/V streams of the
// decode and tile kernels are bounded by the TMA operation rate, profiles/r01b).
kva_status make_pool_map_3d(CUtensorMap *m, void *base, int64_t rows, int d) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (d != 128) return fail(KVA_ERR_UNSUPPORTED, "3-D pool map needs head_dim 128");
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)d * 2, 128};
  cuuint32_t box[3] = {64, 16, 2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed (%d)", (int)r);
  return KVA_OK;
}

// 4-D view {64 channels, 8 rows, 2 halves, row groups} of a d = 128 pool: one box {64, 8, 2, 2}
// is a whole block-head laid out [8-row group][half][8 rows][64] — for a K tile of 8 blocks
// every 8-key group of one half is 2 KB apart, a uniform UMMA stride (SBO = 2048), so the QK
// MMA keeps N = 128 while the K stream needs one TMA operation per block.
kva_status make_pool_map_4d(CUtensorMap *m, void *base, int64_t rows, int d) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (d != 128 || rows % 8) return fail(KVA_ERR_UNSUPPORTED, "4-D pool map needs head_dim 128");
  cuuint64_t dims[4] = {64, 8, 2, (cuuint64_t)(rows / 8)};
  cuuint64_t strides[3] = {(cuuint64_t)d * 2, 128, (cuuint64_t)d * 2 * 8};
  cuuint32_t box[4] = {64, 8, 2, 2};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled (4-D) failed (%d)", (int)r);
  return KVA_OK;
}

kva_status make_pool_map(CUtensorMap *m, void *base, int64_t rows, int d) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (rows >= (1ll << 32)) return fail(KVA_ERR_UNSUPPORTED, "pool has >= 2^32 rows");
  cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)d * 2};
  cuuint32_t box[2] = {64, 16};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KVA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return KVA_OK;
}

}  // namespace

struct kva_pool {
  kva_pool_desc desc;
  std::vector<uint32_t> free_host;  // mirror of free_bits (library is the single writer)
  int64_t n_free = 0;
  CUtensorMap tmk, tmv;
  CUtensorMap tmk3, tmv3;  // 3-D maps (d = 128): one TMA box per block-head
  CUtensorMap tmk4;        // 4-D K map for the tile kernel (N = 128 QK with one box per block)
  bool has3d = false;
  Staging staging;
  // side stream for the tensor-core tile kernel (runs concurrently with the HBM-bound
  // decode kernel on the caller's stream; fork/join by events)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // plan uploads (shared by the pool's plans: a plan created later re-records them, which only
  // orders an earlier plan's run after the later upload as well — never a cycle)
  cudaEvent_t ev_up0 = nullptr, ev_up1 = nullptr;
  // guards the staging ring and the record -> wait -> upload -> record sequence on the shared
  // upload events (calls on one pool must be serialised anyway; this keeps a
  // violation from silently reordering another plan's upload)
  std::mutex up_mu;
  // burst-reserve threshold: < 0 = none
  int64_t threshold_blocks = -1, active_blocks = 0;
};

static int64_t count_free(const std::vector<uint32_t> &w, int nb) {
  int64_t n = 0;
  for (int b = 0; b < nb; ++b) n += (w[b >> 5] >> (b & 31)) & 1u;
  return n;
}

extern "C" kva_status kv_pool_create(const kva_pool_desc *d, kva_pool **out) {
  if (!d || !out) return fail(KVA_ERR_INVALID, "kv_pool_create: null argument");
  *out = nullptr;
  if (d->block_size != kBlock) return fail(KVA_ERR_UNSUPPORTED, "block_size must be 16");
  if (d->head_dim != 64 && d->head_dim != 128)
    return fail(KVA_ERR_UNSUPPORTED, "head_dim must be 64 or 128 (got %d)", d->head_dim);
  if (d->num_blocks <= 0 || d->num_kv_heads <= 0)
    return fail(KVA_ERR_INVALID, "num_blocks and num_kv_heads must be positive");
  if (!d->k_pool || !d->v_pool || !d->free_bits)
    return fail(KVA_ERR_INVALID, "k_pool, v_pool and free_bits are required");
  if ((reinterpret_cast<uintptr_t>(d->k_pool) | reinterpret_cast<uintptr_t>(d->v_pool)) & 127)
    return fail(KVA_ERR_INVALID, "pool tensors must be 128-byte aligned");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (d->device < 0 || d->device >= ndev) return fail(KVA_ERR_INVALID, "bad device %d", d->device);
  DeviceGuard dg(d->device);
  kva_pool *p = new kva_pool();
  p->desc = *d;
  const int words = (d->num_blocks + 31) / 32;
  p->free_host.assign(words, 0);
  cudaError_t e = cudaMemcpy(p->free_host.data(), d->free_bits, words * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    delete p;
    return fail(KVA_ERR_CUDA, "reading free_bits: %s", cudaGetErrorString(e));
  }
  p->n_free = count_free(p->free_host, d->num_blocks);
  {
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&p->aux, cudaStreamNonBlocking, hi) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_up0, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_up1, cudaEventDisableTiming) != cudaSuccess) {
      delete p;
      return fail(KVA_ERR_CUDA, "creating the side stream/events failed");
    }
  }
  const int64_t rows = (int64_t)d->num_blocks * d->num_kv_heads * kBlock;
  kva_status st = make_pool_map(&p->tmk, d->k_pool, rows, d->head_dim);
  if (st == KVA_OK) st = make_pool_map(&p->tmv, d->v_pool, rows, d->head_dim);
  if (st == KVA_OK && d->head_dim == 128) {  // one box per block-head (d = 128 kernels)
    st = make_pool_map_3d(&p->tmk3, d->k_pool, rows, d->head_dim);
    if (st == KVA_OK) st = make_pool_map_4d(&p->tmk4, d->k_pool, rows, d->head_dim);
    if (st == KVA_OK) st = make_pool_map_3d(&p->tmv3, d->v_pool, rows, d->head_dim);
    p->has3d = st == KVA_OK;
  }
  if (st != KVA_OK) {
    delete p;
    return st;
  }
  *out = p;
  return KVA_OK;
}

extern "C" kva_status kv_pool_destroy(kva_pool *p) {
  if (!p) return KVA_OK;
  {
    DeviceGuard dg(p->desc.device);
    p->staging.release();
    if (p->aux) cudaStreamDestroy(p->aux);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->ev_up0) cudaEventDestroy(p->ev_up0);
    if (p->ev_up1) cudaEventDestroy(p->ev_up1);
  }
  delete p;
  return KVA_OK;
}

extern "C" kva_status kv_pool_sync(kva_pool *p, kva_stream_t stream) {
  (void)stream;  // every kv_append write is on the caller's stream: nothing to order
  if (!p) return fail(KVA_ERR_INVALID, "null pool");
  return KVA_OK;
}

extern "C" kva_status kv_pool_free_count(const kva_pool *p, int64_t *n) {
  if (!p || !n) return fail(KVA_ERR_INVALID, "null argument");
  *n = p->n_free;
  return KVA_OK;
}

extern "C" kva_status kv_pool_resync(kva_pool *p) {
  if (!p) return fail(KVA_ERR_INVALID, "null pool");
  DeviceGuard dg(p->desc.device);
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(p->free_host.data(), p->desc.free_bits, p->free_host.size() * 4,
                      cudaMemcpyDeviceToHost));
  p->n_free = count_free(p->free_host, p->desc.num_blocks);
  return KVA_OK;
}

// ------------------------------------------------------------------------------------------
// descriptor validation (host, synchronous, before anything is enqueued)
// ------------------------------------------------------------------------------------------
static inline int qlen(const kva_batch_desc *b, int i) { return b->q_indptr[i + 1] - b->q_indptr[i]; }
static inline int cdiv(int a, int b) { return (a + b - 1) / b; }

// mode 0: attention (every block of [0, ctx) allocated); mode 1: append (resident part only)
static kva_status validate_batch(const kva_batch_desc *b, int nb, int mode) {
  if (!b) return fail(KVA_ERR_INVALID, "null descriptor");
  if (b->num_reqs < 0) return fail(KVA_ERR_INVALID, "num_reqs < 0");
  if (b->head_dim != 64 && b->head_dim != 128)
    return fail(KVA_ERR_UNSUPPORTED, "head_dim must be 64 or 128 (got %d)", b->head_dim);
  if (b->num_kv_heads <= 0) return fail(KVA_ERR_INVALID, "num_kv_heads <= 0");
  if (b->num_q_heads <= 0 || b->num_q_heads % b->num_kv_heads)
    return fail(KVA_ERR_INVALID, "num_q_heads %d not a positive multiple of num_kv_heads %d",
                b->num_q_heads, b->num_kv_heads);
  if (b->num_reqs == 0) return KVA_OK;
  if (!b->q_indptr || !b->ctx_len || !b->block_table || !b->block_table_host)
    return fail(KVA_ERR_INVALID, "q_indptr, ctx_len, block_table and block_table_host are required");
  if (b->max_blocks <= 0) return fail(KVA_ERR_INVALID, "max_blocks <= 0");
  if (b->q_indptr[0] != 0) return fail(KVA_ERR_INVALID, "q_indptr[0] != 0");
  // a group member's prefix entries equal its group's first member's (checked below, entry by
  // entry), so only the first member of each group range-checks them
  const int Gv = b->group_of ? std::max(b->num_groups, 0) : 0;
  std::vector<int> first_of(Gv, -1);
  for (int i = 0; i < b->num_reqs && Gv > 0; ++i) {
    const int gi = b->group_of[i];
    if (gi >= 0 && gi < Gv && first_of[gi] < 0) first_of[gi] = i;
  }
  for (int i = 0; i < b->num_reqs; ++i) {
    const int ql = qlen(b, i), ctx = b->ctx_len[i];
    if (ql < 1 || ql > ctx) return fail(KVA_ERR_INVALID, "request %d: q_len %d not in [1, ctx=%d]", i, ql, ctx);
    if (ctx > b->max_blocks * kBlock)
      return fail(KVA_ERR_INVALID, "request %d: ctx %d > max_blocks*16", i, ctx);
    const int need_blocks = mode == 0 ? cdiv(ctx, kBlock) : cdiv(ctx - ql, kBlock);
    const int32_t *row = b->block_table_host + (int64_t)i * b->max_blocks;
    const int gi = Gv > 0 ? b->group_of[i] : -1;
    const int k0 = (gi >= 0 && gi < Gv && first_of[gi] != i && b->group_prefix_blocks)
                       ? std::max(0, std::min(b->group_prefix_blocks[gi], need_blocks)) : 0;
    uint32_t bad = 0;  // branch-free (vectorised) range check; the slow path names the entry
    for (int k = k0; k < need_blocks; ++k) bad |= (uint32_t)row[k] >= (uint32_t)nb;
    if (bad)
      for (int k = 0; k < need_blocks; ++k)
        if (row[k] < 0 || row[k] >= nb)
          return fail(KVA_ERR_INVALID, "request %d: block_table[%d] = %d invalid (num_blocks %d)", i, k,
                      row[k], nb);
  }
  if (b->group_of) {
    const int G = std::max(b->num_groups, 0);
    if (G > 0 && !b->group_prefix_blocks)
      return fail(KVA_ERR_INVALID, "group_prefix_blocks required");
    for (int gi = 0; gi < G; ++gi) {
      if (b->group_prefix_blocks[gi] < 0) return fail(KVA_ERR_GROUP, "group %d: negative prefix", gi);
      if (!b->group_parent) continue;
      const int pa = b->group_parent[gi];
      if (pa < -1 || pa >= gi) return fail(KVA_ERR_GROUP, "group %d: parent %d not an earlier group", gi, pa);
      if (pa >= 0 && b->group_prefix_blocks[pa] > b->group_prefix_blocks[gi])
        return fail(KVA_ERR_GROUP, "group %d: shorter prefix than its parent %d", gi, pa);
      int depth = 1;
      for (int x = pa; x >= 0; x = b->group_parent[x]) ++depth;
      if (depth > kMaxCascade) return fail(KVA_ERR_UNSUPPORTED, "group %d: nesting deeper than %d", gi, kMaxCascade);
    }
    std::vector<int> first(G, -1);  // first request whose chain contains the group
    for (int i = 0; i < b->num_reqs; ++i) {
      const int gi = b->group_of[i];
      if (gi < 0) continue;
      if (gi >= G) return fail(KVA_ERR_GROUP, "request %d: group %d out of range", i, gi);
      const int np = b->group_prefix_blocks[gi];
      if (b->ctx_len[i] - qlen(b, i) < np * kBlock)
        return fail(KVA_ERR_GROUP, "request %d: queries/appends inside group %d's prefix", i, gi);
      const int32_t *a = b->block_table_host + (int64_t)i * b->max_blocks;
      // every level of the chain: the first n_l entries equal the level's blocks
      // (entries are in range: the prefix lies inside the resident part checked above)
      for (int l = gi; l >= 0; l = b->group_parent ? b->group_parent[l] : -1) {
        if (first[l] < 0) first[l] = i;
        const int32_t *c = b->block_table_host + (int64_t)first[l] * b->max_blocks;
        const int nl = b->group_prefix_blocks[l];
        if (std::memcmp(a, c, (size_t)nl * sizeof(int32_t)) != 0)
          for (int k = 0; k < nl; ++k)
            if (a[k] != c[k])
              return fail(KVA_ERR_GROUP, "request %d: prefix block %d differs from group %d's", i, k, l);
      }
    }
  }
  return KVA_OK;
}

static kva_status validate_desc(const kva_pool *p, const kva_batch_desc *b, int mode) {
  if (!p || !b) return fail(KVA_ERR_INVALID, "null pool or descriptor");
  if (b->num_kv_heads != p->desc.num_kv_heads)
    return fail(KVA_ERR_INVALID, "num_kv_heads %d != pool's %d", b->num_kv_heads, p->desc.num_kv_heads);
  if (b->head_dim != p->desc.head_dim)
    return fail(KVA_ERR_INVALID, "head_dim %d != pool's %d", b->head_dim, p->desc.head_dim);
  return validate_batch(b, p->desc.num_blocks, mode);
}

extern "C" kva_status kva_validate_batch(const kva_batch_desc *b, int32_t num_blocks, int32_t mode) {
  if (mode != 0 && mode != 1) return fail(KVA_ERR_INVALID, "mode must be 0 or 1");
  return validate_batch(b, num_blocks, mode);
}

// ------------------------------------------------------------------------------------------
// kv_append (a2)
// ------------------------------------------------------------------------------------------
struct AppendPlan {
  std::vector<int32_t> tbl_idx, ids;
  int64_t need = 0;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t append_upload_bytes(int R, int64_t nalloc) {  // both request lists + allocations
  return 2 * align256(sizeof(AppendReq) * std::max(R, 1)) + 2 * align256(4 * (R + 1)) +
         2 * align256(4 * std::max<int64_t>(nalloc, 1));
}

extern "C" kva_status kv_append_workspace_size(const kva_batch_desc *b, size_t *bytes) {
  if (!b || !bytes) return fail(KVA_ERR_INVALID, "null argument");
  // the same descriptor checks kv_append runs (any block id passes: no pool here)
  if (kva_status st = validate_batch(b, INT32_MAX, 1); st != KVA_OK) return st;
  // upper bound on allocations: every new position's block
  int64_t nalloc = 0;
  for (int i = 0; i < b->num_reqs; ++i) {
    const int ql = qlen(b, i), ctx = b->ctx_len[i];
    nalloc += cdiv(ctx, kBlock) - (ctx - ql) / kBlock;
  }
  *bytes = append_upload_bytes(b->num_reqs, nalloc);
  return KVA_OK;
}

// validated: the caller has just run validate_desc(p, b, 1) (kv_append_plan)
static kva_status append_impl(kva_pool *p, kva_batch_desc *b, const void *k_new, const void *v_new,
                              int64_t stride_tok, int32_t *deficit, void *workspace, size_t ws_bytes,
                              kva_stream_t stream, bool validated) {
  if (deficit) *deficit = 0;
  HSection hs;
  kva_status st = validated ? KVA_OK : validate_desc(p, b, 1);
  hs.lap("append.validate");
  if (st != KVA_OK) return st;
  if (b->num_reqs == 0) return KVA_OK;
  const int Hkv = b->num_kv_heads, d = b->head_dim, nb = p->desc.num_blocks;
  if (!k_new || !v_new) return fail(KVA_ERR_INVALID, "k_new/v_new required");
  if (stride_tok < (int64_t)Hkv * d) return fail(KVA_ERR_INVALID, "new_stride_tok too small");
  if (((reinterpret_cast<uintptr_t>(k_new) | reinterpret_cast<uintptr_t>(v_new)) & 15) ||
      (stride_tok % 8))
    return fail(KVA_ERR_INVALID, "k_new/v_new must be 16-byte aligned with stride %% 8 == 0");
  AppendPlan ap;
  int64_t need_offline = 0;
  // count needed blocks (entries == -1 among new positions' blocks), validate the rest
  for (int i = 0; i < b->num_reqs; ++i) {
    const int64_t need_before = ap.need;
    const int ql = qlen(b, i), ctx = b->ctx_len[i], start = ctx - ql;
    if (cdiv(ctx, kBlock) > nb)
      return fail(KVA_ERR_CAPACITY, "request %d needs %d blocks > pool's %d", i, cdiv(ctx, kBlock), nb);
    const int32_t *row = b->block_table_host + (int64_t)i * b->max_blocks;
    for (int k = start / kBlock; k < cdiv(ctx, kBlock); ++k) {
      if (row[k] == -1) ++ap.need;
      else if (row[k] < 0 || row[k] >= nb)
        return fail(KVA_ERR_INVALID, "request %d: block_table[%d] = %d invalid", i, k, row[k]);
    }
    const int32_t ty = b->req_type ? b->req_type[i] : KVA_ONLINE_DECODE;
    if (ty == KVA_OFFLINE_PREFILL || ty == KVA_OFFLINE_DECODE) need_offline += ap.need - need_before;
  }
  if (ap.need > p->n_free) {
    if (deficit) *deficit = (int32_t)(ap.need - p->n_free);
    return fail(KVA_NEEDS_EVICTION, "kv_append needs %lld blocks, %lld free", (long long)ap.need,
                (long long)p->n_free);
  }
  // burst reserve: offline allocations may not push the active classes over the threshold;
  // online ones may use the reserve (reading R35)
  if (p->threshold_blocks >= 0 && need_offline > 0 && p->active_blocks + ap.need > p->threshold_blocks) {
    if (deficit) *deficit = (int32_t)(p->active_blocks + ap.need - p->threshold_blocks);
    return fail(KVA_NEEDS_EVICTION, "kv_append: %lld active + %lld new blocks > threshold %lld",
                (long long)p->active_blocks, (long long)ap.need, (long long)p->threshold_blocks);
  }
  const size_t up = append_upload_bytes(b->num_reqs, ap.need);
  if (!workspace || ws_bytes < up)
    return fail(KVA_ERR_INVALID, "kv_append workspace too small (%zu < %zu)", ws_bytes, up);
  // allocate: descriptor order, positions ascending, smallest free id first (reading #13)
  hs.lap("append.count");
  std::vector<uint32_t> fh = p->free_host;  // commit only after everything is enqueued
  std::vector<int32_t> first_new(b->num_reqs);  // request i's allocations: ap.ids[first_new[i] ...]
  int scan = 0;
  for (int i = 0; i < b->num_reqs; ++i) {
    first_new[i] = (int32_t)ap.ids.size();
    const int ql = qlen(b, i), ctx = b->ctx_len[i], start = ctx - ql;
    const int32_t *row = b->block_table_host + (int64_t)i * b->max_blocks;
    for (int k = start / kBlock; k < cdiv(ctx, kBlock); ++k) {
      if (row[k] != -1) continue;
      while (!((fh[scan >> 5] >> (scan & 31)) & 1u)) ++scan;
      fh[scan >> 5] &= ~(1u << (scan & 31));
      ap.tbl_idx.push_back(i * b->max_blocks + k);
      ap.ids.push_back(scan);
    }
  }
  hs.lap("append.alloc");
  DeviceGuard dg(p->desc.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  hs.lap("append.guard");
  // Two request lists: decode-class requests (<= 16 rows: their <= 2 blocks resolved here, so
  // their append reads no table entry and shares one launch with the allocation publishing),
  // then the rest (prefill chunks, whose rows are read only by the tile kernel: that launch
  // reads the freshly written table and lets the tile kernel start early, PDL).  Lists travel
  // as kernel parameters unless they overflow the inline capacity.
  const int g = b->num_q_heads / b->num_kv_heads;
  std::vector<AppendReq> ra, rb;
  std::vector<int32_t> pa{0}, pbv{0};
  for (int i = 0; i < b->num_reqs; ++i) {
    const int ql = qlen(b, i);
    if (ql == 0) continue;
    AppendReq rq{b->q_indptr[i], ql, b->ctx_len[i] - ql, i, {-1, -1}};
    if (ql * g <= kDecodeRows) {
      const int32_t *row = b->block_table_host + (int64_t)i * b->max_blocks;
      int cur = first_new[i];
      const int kb0 = rq.pos0 / kBlock, kb1 = cdiv(b->ctx_len[i], kBlock);
      for (int k = kb0; k < kb1 && k < kb0 + 2; ++k) rq.blk[k - kb0] = row[k] != -1 ? row[k] : ap.ids[cur++];
      ra.push_back(rq);
      pa.push_back(pa.back() + ql);
    } else {
      rb.push_back(rq);
      pbv.push_back(pbv.back() + ql);
    }
  }
  ReqList<AppendReq> la{}, lb{};
  AllocList al{};
  la.n = (int32_t)ra.size();
  lb.n = (int32_t)rb.size();
  al.n = (int32_t)ap.ids.size();
  const bool up_a = ra.size() > (size_t)kInlineReqs, up_b = rb.size() > (size_t)kInlineReqs;
  const bool up_al = ap.ids.size() > (size_t)kInlineAlloc;
  if (!up_a) {
    std::copy(ra.begin(), ra.end(), la.req);
    std::copy(pa.begin(), pa.end(), la.pre);
  }
  if (!up_b) {
    std::copy(rb.begin(), rb.end(), lb.req);
    std::copy(pbv.begin(), pbv.end(), lb.pre);
  }
  if (!up_al) {
    std::copy(ap.tbl_idx.begin(), ap.tbl_idx.end(), al.tbl);
    std::copy(ap.ids.begin(), ap.ids.end(), al.ids);
  }
  if (up_a || up_b || up_al) {
    std::lock_guard<std::mutex> lk(p->up_mu);
    Staging::Slot *slot = nullptr;
    CUDA_TRY(p->staging.get(up, &slot));
    uint8_t *h = static_cast<uint8_t *>(slot->host);
    uint8_t *dws = static_cast<uint8_t *>(workspace);
    size_t off = 0;
    auto put = [&](const void *src, size_t n) {
      if (n) std::memcpy(h + off, src, n);
      const size_t o = off;
      off += align256(std::max<size_t>(n, 4));
      return dws + o;
    };
    if (up_a) {
      la.ptr = reinterpret_cast<const AppendReq *>(put(ra.data(), sizeof(AppendReq) * ra.size()));
      la.pre_ptr = reinterpret_cast<const int32_t *>(put(pa.data(), 4 * pa.size()));
    }
    if (up_b) {
      lb.ptr = reinterpret_cast<const AppendReq *>(put(rb.data(), sizeof(AppendReq) * rb.size()));
      lb.pre_ptr = reinterpret_cast<const int32_t *>(put(pbv.data(), 4 * pbv.size()));
    }
    if (up_al) {
      al.tbl_ptr = reinterpret_cast<const int32_t *>(put(ap.tbl_idx.data(), 4 * ap.tbl_idx.size()));
      al.ids_ptr = reinterpret_cast<const int32_t *>(put(ap.ids.data(), 4 * ap.ids.size()));
    }
    CUDA_TRY(p->staging.upload(slot, workspace, off, s));
  }
  hs.lap("append.lists");
  uint16_t *kp = static_cast<uint16_t *>(p->desc.k_pool), *vp = static_cast<uint16_t *>(p->desc.v_pool);
  const uint16_t *kn = static_cast<const uint16_t *>(k_new), *vn = static_cast<const uint16_t *>(v_new);
  // the decode-class append lets the prefill-row append (which waits for it) be set up early;
  // with no prefill rows the attention follows it directly and it must complete first
  CUDA_TRY(launch_append(kn, vn, stride_tok, kp, vp, Hkv, d, b->block_table, b->max_blocks, la, pa.back(), s,
                         /*early_trigger=*/!rb.empty(), &al, p->desc.free_bits));
  if (!rb.empty())  // the tile kernel (PDL) may start while these rows are written
    CUDA_TRY(launch_append(kn, vn, stride_tok, kp, vp, Hkv, d, b->block_table, b->max_blocks, lb, pbv.back(), s,
                           /*early_trigger=*/true));
  hs.lap("append.launch_append");
  p->active_blocks += ap.need;  // every new block belongs to a running request
  // commit host state: free mirror + caller's host table mirror
  p->free_host.swap(fh);
  p->n_free -= ap.need;
  for (size_t j = 0; j < ap.ids.size(); ++j) b->block_table_host[ap.tbl_idx[j]] = ap.ids[j];
  hs.lap("append.commit");
  return KVA_OK;
}

extern "C" kva_status kv_append(kva_pool *p, kva_batch_desc *b, const void *k_new,
                                const void *v_new, int64_t stride_tok, int32_t *deficit,
                                void *workspace, size_t ws_bytes, kva_stream_t stream) {
  return append_impl(p, b, k_new, v_new, stride_tok, deficit, workspace, ws_bytes, stream, false);
}

// ------------------------------------------------------------------------------------------
// hybrid attention planner (a1)
// ------------------------------------------------------------------------------------------
struct kva_plan {
  AttnParams p;
  CUtensorMap tmk, tmv;
  CUtensorMap tmk3, tmv3, tmk4;
  bool has3d = false;
  ReqList<DecodeReq> dec;                  // decode requests (inline kernel parameter or uploaded)
  ReqList<MergeReq> mrg;                   // merged requests (idem)
  ReqList<MergeReq> mrg_red;               // the same without the folded requests (fold mode)
  int n_mrows_red = 0;
  bool has_fold = false;                   // FoldReq list + counters in the workspace
  mutable uint32_t runs = 0;               // runs that launched the tile kernel (fold epoch)
  TileList tiles;                          // tcgen05 tile items (inline kernel parameter or uploaded)
  int n_dec = 0, n_tile = 0, n_mrows = 0;  // work units: decode (split, head), tiles, merge (row, head)
  // the plan arrays are uploaded on the pool's side stream (ordered after `stream`'s prior work
  // by ev_up0); a kernel that reads uploaded arrays on `stream` first waits ev_up1 (both owned
  // by the pool)
  cudaEvent_t ev_up0 = nullptr, ev_up1 = nullptr;
  bool uploaded = false;
  kva_pool *pool = nullptr;  // for the side-stream append event (the pool outlives its plans)
  int device = 0;
  int tile_ctas = 0;              // persistent tile-kernel grid (0 = all SMs)
  bool overlap = true;            // tile kernel on the side stream, concurrent with decode
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t t_ev[4] = {nullptr, nullptr, nullptr, nullptr};  // optional timing events
  unsigned long long *span = nullptr;                           // optional in-kernel spans
  int n_out_extra = 0;                                          // fused a7: peer destinations
  void *out_extra[kMaxOutExtra] = {};
  kva_plan_stats stats{};
};

struct PlanBuild {
  std::vector<DecodeReq> dec;
  std::vector<int32_t> dec_pre{0};   // exclusive prefix of splits per decode request
  std::vector<TileItem> tile;
  std::vector<MergeReq> mrg;
  std::vector<int32_t> mrg_pre{0};   // exclusive prefix of rows per merged request
  std::vector<int32_t> row_list;
  std::vector<FoldReq> fold;          // folded decode-class members (DecodeReq::fold)
  std::vector<MergeReq> mrg_red;      // the merge list without them (fold mode)
  std::vector<int32_t> mrg_red_pre{0};
  int32_t n_casc_items = 0;           // cascade tile items (fold counters: 2 per item)
  int64_t n_slots = 0;
  int64_t tile_flops = 0;
  kva_plan_stats stats{};
};

static void build_plan(const kva_batch_desc *b, PlanBuild &pb) {
  HSection hb;
  const int kTileM = 2 * kTileMTc;  // rows per tile item: the tcgen05 kernel's two Q tiles
  const int R = b->num_reqs, Hkv = b->num_kv_heads, Hq = b->num_q_heads, g = Hq / Hkv;
  const int d = b->head_dim;
  const int G = b->group_of ? std::max(b->num_groups, 0) : 0;
  auto grp = [&](int i) { return b->group_of ? b->group_of[i] : -1; };
  auto dec_class = [&](int i) { return qlen(b, i) * g <= kDecodeRows; };
  // --- cascade tiles: decode-class members of each group, stacked along M; a nested group
  // (level) covers keys [n_parent*16, n_g*16) and stacks every member at or below it ---
  auto parent = [&](int gi) { return b->group_parent ? b->group_parent[gi] : -1; };
  auto in_chain = [&](int i, int gi) {
    for (int l = grp(i); l >= 0; l = parent(l))
      if (l == gi) return true;
    return false;
  };
  std::vector<int> first_member(G, -1);
  std::vector<std::vector<int>> members(G);  // decode-class requests at or below the group
  std::vector<std::vector<int>> member_off(G);  // their token offsets in the group's row list
  std::vector<int64_t> casc_base(G, -1);
  std::vector<int> group_rows(G, 0), list_off(G, 0), flag_base(G, -1), mtiles(G, 0);
  for (int i = 0; i < R; ++i)
    for (int l = grp(i); l >= 0; l = parent(l))
      if (first_member[l] < 0) first_member[l] = i;
  for (int gi = 0; gi < G; ++gi) {
    list_off[gi] = (int)pb.row_list.size();
    for (int i = 0; i < R; ++i) {
      if (grp(i) < 0 || !dec_class(i) || !in_chain(i, gi)) continue;
      members[gi].push_back(i);
      member_off[gi].push_back((int)pb.row_list.size() - list_off[gi]);
      for (int j = 0; j < qlen(b, i); ++j) pb.row_list.push_back(b->q_indptr[i] + j);
    }
    const int ntok = (int)pb.row_list.size() - list_off[gi];
    group_rows[gi] = ntok * g;
    if (ntok == 0) continue;
    const int np = b->group_prefix_blocks[gi];
    const int kstart = parent(gi) >= 0 ? b->group_prefix_blocks[parent(gi)] * kBlock : 0;
    casc_base[gi] = pb.n_slots;
    if (np * kBlock > kstart) {  // cascade item (gi, h, m0) = flag_base + h * mtiles + m0 / kTileM
      flag_base[gi] = pb.n_casc_items;
      mtiles[gi] = cdiv(group_rows[gi], kTileM);
      pb.n_casc_items += Hkv * mtiles[gi];
    }
    for (int h = 0; h < Hkv; ++h) {
      for (int m0 = 0; m0 < group_rows[gi]; m0 += kTileM) {
        if (np * kBlock <= kstart) break;  // a level with no blocks of its own: no tile
        TileItem t{};
        t.row_src = list_off[gi];
        t.r0 = m0;
        t.n_rows = std::min(kTileM, group_rows[gi] - m0);
        t.kv_head = h;
        t.table_row = first_member[gi];
        t.k0 = kstart;
        t.k1 = np * kBlock;
        t.pos0 = 0;
        t.slot = (int32_t)(pb.n_slots + m0);
        t.flags = kTileList | ((flag_base[gi] + h * mtiles[gi] + m0 / kTileM + 1) << 8);
        pb.tile.push_back(t);
        pb.stats.n_cascade_items++;
      }
      pb.n_slots += group_rows[gi];
    }
  }
  hb.lap("build.cascade");
  // the merge lists a level only if it has a tile (blocks of its own)
  auto level_has_tile = [&](int gi) {
    const int kstart = parent(gi) >= 0 ? b->group_prefix_blocks[parent(gi)] * kBlock : 0;
    return b->group_prefix_blocks[gi] * kBlock > kstart;
  };
  // --- per request ---
  {
    size_t nd = 0, nm = 0;
    for (int i = 0; i < R; ++i)
      if (dec_class(i)) {
        ++nd;
        ++nm;
      }
    pb.dec.reserve(nd);
    pb.dec_pre.reserve(nd + 1);
    pb.mrg.reserve(nm);
    pb.mrg_pre.reserve(nm + 1);
    pb.mrg_red.reserve(nm);
    pb.mrg_red_pre.reserve(nm + 1);
    pb.fold.reserve(nm);
  }
  // a member's position in its level's member list: the members are listed in request order,
  // so a running cursor per level replaces the binary search
  std::vector<int> cursor(G, 0);
  int64_t kv_tokens = 0, dec_keys = 0, dec_rows = 0;
  for (int gi = 0; gi < G; ++gi)  // each level's own blocks once
    kv_tokens += (int64_t)(b->group_prefix_blocks[gi] - (parent(gi) >= 0 ? b->group_prefix_blocks[parent(gi)] : 0)) * kBlock;
  for (int i = 0; i < R; ++i) {
    const int ql = qlen(b, i), ctx = b->ctx_len[i], gi = grp(i), q0 = b->q_indptr[i];
    const int np = gi >= 0 ? b->group_prefix_blocks[gi] : 0;
    kv_tokens += ctx - np * kBlock;
    // sum_{j<ql} (ctx - ql + j + 1) visible keys per q-head
    pb.stats.flops += ((int64_t)ql * (ctx - ql + 1) + (int64_t)ql * (ql - 1) / 2) * Hq * 4 * d;
    if (dec_class(i)) {
      const bool cascaded = gi >= 0;
      const int kb = cascaded ? np * kBlock : 0;
      const int nsplit = cdiv(ctx - kb, kSplitKeys);
      const bool direct = !cascaded && nsplit == 1;
      const int rows = ql * g;
      dec_rows += rows * Hkv;
      // head-factored: one request entry; the kernel runs every (split, kv head); partial slot
      // of (head h, split s, row r) = base + (h * nsplit + s) * rows + r
      const int64_t base = direct ? -1 : pb.n_slots;
      if (!direct) pb.n_slots += (int64_t)nsplit * rows * Hkv;
      DecodeReq dq{};
      dq.q_row0 = q0;
      dq.n_tok = ql;
      dq.table_row = i;
      dq.kb = kb;
      dq.ctx = ctx;
      dq.slot = direct ? -1 : (int32_t)base;
      dq.nsplit = nsplit;
      dq.fold = -1;
      pb.dec.push_back(dq);
      pb.dec_pre.push_back(pb.dec_pre.back() + nsplit);
      dec_keys += (int64_t)(ctx - kb) * Hkv;
      if (!direct) {
        MergeReq mq{};
        mq.q_row0 = q0;
        mq.rows = rows;
        mq.n_casc = 0;
        // level l's partial of (head h, row r): casc_base[l] + h * group_rows[l] + off * g + r
        int pos0 = 0;  // position in the deepest level's member list
        for (int l = cascaded ? gi : -1; l >= 0; l = parent(l)) {
          const auto &mv = members[l];
          int &cur = cursor[l];
          while (cur < (int)mv.size() && mv[cur] < i) ++cur;  // members[l] is ascending
          const int pos = cur;
          if (l == gi) pos0 = pos;
          if (!level_has_tile(l)) continue;
          mq.casc_slot[mq.n_casc] = (int32_t)(casc_base[l] + (int64_t)member_off[l][pos] * g);
          mq.casc_hstride[mq.n_casc] = group_rows[l];
          ++mq.n_casc;
        }
        mq.split_slot = (int32_t)base;
        mq.nsplit = nsplit;
        pb.mrg.push_back(mq);
        pb.mrg_pre.push_back(pb.mrg_pre.back() + rows);
        // fold: a member of a one-level group whose suffix is one split (the decode warp owns
        // the whole suffix partial and merges it with the cascade partial itself)
        if (cascaded && parent(gi) < 0 && level_has_tile(gi) && nsplit == 1 && mq.n_casc == 1) {
          FoldReq fr{};
          fr.casc_slot = mq.casc_slot[0];
          fr.casc_hstride = mq.casc_hstride[0];
          fr.member_row0 = member_off[gi][pos0] * g;
          fr.flag_base = flag_base[gi];
          fr.mtiles = mtiles[gi];
          pb.dec.back().fold = (int32_t)pb.fold.size();  // (dq was pushed above)
          pb.fold.push_back(fr);
        } else {
          pb.mrg_red.push_back(mq);
          pb.mrg_red_pre.push_back(pb.mrg_red_pre.back() + rows);
        }
      }
    } else {
      const int rows = ql * g;
      for (int h = 0; h < Hkv; ++h) {
        for (int m0 = 0; m0 < rows; m0 += kTileM) {
          TileItem t{};
          t.row_src = q0;
          t.r0 = m0;
          t.n_rows = std::min(kTileM, rows - m0);
          t.kv_head = h;
          t.table_row = i;
          t.k0 = 0;
          t.k1 = ctx - ql + (m0 + t.n_rows - 1) / g + 1;
          t.pos0 = ctx - ql;
          t.slot = -1;
          t.flags = kTileCausal;
          pb.tile.push_back(t);
        }
      }
    }
  }
  hb.lap("build.requests");
  // longest tiles first (LPT); ties keep (kv_head, m-tile, member) order so concurrently
  // running CTAs of a group share its prefix blocks in L2
  // F(x) = sum_{r<x} floor(r/g) (closed form), so a causal tile's visible keys are exact
  auto F = [g](int64_t x) { const int64_t q = x / g; return g * q * (q - 1) / 2 + q * (x - q * g); };
  for (const TileItem &t : pb.tile) {
    if (t.flags & kTileCausal) {  // row r sees keys [0, pos0 + r/g]
      const int64_t keys = (int64_t)t.n_rows * (t.pos0 + 1) + F(t.r0 + t.n_rows) - F(t.r0);
      pb.stats.tile_flops += keys * 4 * d;
    } else {
      pb.stats.tile_flops += (int64_t)t.n_rows * (t.k1 - t.k0) * 4 * d;
    }
  }
  pb.tile_flops = pb.stats.tile_flops;
  std::stable_sort(pb.tile.begin(), pb.tile.end(),
                   [](const TileItem &a, const TileItem &c) { return a.k1 - a.k0 > c.k1 - c.k0; });
  // decode requests longest first (LPT): the decode grid runs ~1.7 waves (2 CTAs/SM by shared
  // memory), and a short request's CTAs then fill the tail instead of a long one's; each
  // request keeps its partial slots, so the order changes no arithmetic
  {
    std::vector<int> ord(pb.dec.size());
    for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) {
      return pb.dec[x].ctx - pb.dec[x].kb > pb.dec[y].ctx - pb.dec[y].kb;
    });
    std::vector<DecodeReq> dec(pb.dec.size());
    std::vector<int32_t> pre(pb.dec.size() + 1, 0);
    for (size_t i = 0; i < ord.size(); ++i) {
      dec[i] = pb.dec[ord[i]];
      pre[i + 1] = pre[i] + dec[i].nsplit;
    }
    pb.dec.swap(dec);
    pb.dec_pre.swap(pre);
  }
  hb.lap("build.sort");
  pb.stats.n_decode_items = (int64_t)pb.dec_pre.back() * Hkv;  // (split, head) units
  pb.stats.n_tile_items = (int64_t)pb.tile.size();
  pb.stats.n_merge_rows = (int64_t)pb.mrg_pre.back() * Hkv;
  pb.stats.kv_bytes_algorithmic = kv_tokens * Hkv * d * 2 * 2;
  const int64_t total_q = b->q_indptr[R];
  pb.stats.q_bytes = total_q * Hq * d * 2;
  pb.stats.o_bytes = total_q * Hq * d * 2;
  pb.stats.decode_kv_bytes = dec_keys * d * 2 * 2;
  (void)dec_rows;
}

static size_t plan_bytes(const PlanBuild &pb, int d, size_t *arrays_bytes) {
  // upper bound: the request lists count even when they travel as kernel parameters
  size_t a = align256(sizeof(DecodeReq) * pb.dec.size()) + align256(4 * pb.dec_pre.size()) +
             align256(sizeof(MergeReq) * pb.mrg.size()) + align256(4 * pb.mrg_pre.size()) +
             align256(sizeof(TileItem) * pb.tile.size()) + align256(4 * pb.row_list.size()) +
             align256(sizeof(MergeReq) * pb.mrg_red.size()) + align256(4 * pb.mrg_red_pre.size()) +
             align256(sizeof(FoldReq) * pb.fold.size()) + align256(8 * (size_t)pb.n_casc_items) + 10 * 256;
  if (arrays_bytes) *arrays_bytes = a;
  return a + align256((size_t)pb.n_slots * d * 4) + align256((size_t)pb.n_slots * 4);
}

extern "C" kva_status hybrid_attention_workspace_size(const kva_batch_desc *b, size_t *bytes) {
  if (!b || !bytes) return fail(KVA_ERR_INVALID, "null argument");
  // build_plan walks group chains and indexes per-group arrays: the descriptor is validated
  // first (groups, parents, shapes; the table's unallocated new-position entries may be -1)
  if (kva_status st = validate_batch(b, INT32_MAX, 1); st != KVA_OK) return st;
  PlanBuild pb;
  build_plan(b, pb);
  *bytes = plan_bytes(pb, b->head_dim, nullptr);
  return KVA_OK;
}

// validated = the caller has just validated the descriptor for attention (kv_append_plan:
// kv_append checked the resident part and filled every new position's entry itself)
static kva_status plan_impl(kva_pool *p, const kva_batch_desc *b, void *ws, size_t ws_bytes,
                            kva_stream_t stream, kva_plan **out, bool validated) {
  if (!out) return fail(KVA_ERR_INVALID, "null plan pointer");
  *out = nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  HSection hs;
  kva_status st = validated ? KVA_OK : validate_desc(p, b, 0);
  hs.lap("plan.validate");
  if (st != KVA_OK) return st;
  const auto t1 = std::chrono::steady_clock::now();
  PlanBuild pb;
  build_plan(b, pb);
  const auto t2 = std::chrono::steady_clock::now();
  hs.lap("plan.build");
  size_t arrays = 0;
  const size_t need = plan_bytes(pb, b->head_dim, &arrays);
  if (!ws || ws_bytes < need)
    return fail(KVA_ERR_INVALID, "hybrid_attention workspace too small (%zu < %zu)", ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(KVA_ERR_INVALID, "workspace must be 256-B aligned");
  DeviceGuard dg(p->desc.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  hs.lap("plan.guard");
  kva_plan *pl = new kva_plan();
  hs.lap("plan.new");
  pl->device = p->desc.device;
  pl->tmk = p->tmk;
  pl->tmv = p->tmv;
  pl->tmk3 = p->tmk3;
  pl->tmk4 = p->tmk4;
  pl->tmv3 = p->tmv3;
  pl->has3d = p->has3d;
  pl->stats = pb.stats;
  uint8_t *dws = static_cast<uint8_t *>(ws);
  // request lists: kernel parameters when they fit, else uploaded with the tile items
  const bool dec_inline = pb.dec.size() <= (size_t)kInlineReqs;
  const bool mrg_inline = pb.mrg.size() <= (size_t)kInlineReqs;
  pl->dec.n = (int32_t)pb.dec.size();
  pl->mrg.n = (int32_t)pb.mrg.size();
  if (dec_inline) {
    std::copy(pb.dec.begin(), pb.dec.end(), pl->dec.req);
    std::copy(pb.dec_pre.begin(), pb.dec_pre.end(), pl->dec.pre);
  }
  if (mrg_inline) {
    std::copy(pb.mrg.begin(), pb.mrg.end(), pl->mrg.req);
    std::copy(pb.mrg_pre.begin(), pb.mrg_pre.end(), pl->mrg.pre);
  }
  const bool has_fold = !pb.fold.empty();
  const bool mrg_red_inline = pb.mrg_red.size() <= (size_t)kInlineReqs;
  pl->mrg_red.n = (int32_t)pb.mrg_red.size();
  if (has_fold && mrg_red_inline) {
    std::copy(pb.mrg_red.begin(), pb.mrg_red.end(), pl->mrg_red.req);
    std::copy(pb.mrg_red_pre.begin(), pb.mrg_red_pre.end(), pl->mrg_red.pre);
  }
  const bool tile_inline = pb.tile.size() <= (size_t)kInlineTiles;
  pl->tiles.n = (int32_t)pb.tile.size();
  pl->tiles.ptr = nullptr;
  if (tile_inline) std::copy(pb.tile.begin(), pb.tile.end(), pl->tiles.item);
  const bool need_upload = (!pb.tile.empty() && !tile_inline) || !pb.row_list.empty() || !dec_inline || !mrg_inline ||
                           has_fold;
  hs.lap("plan.inline_copy");
  if (need_upload) {
    std::lock_guard<std::mutex> lk(p->up_mu);
    Staging::Slot *slot = nullptr;
    cudaError_t e = p->staging.get(arrays, &slot);
    if (e != cudaSuccess) {
      delete pl;
      return fail(KVA_ERR_CUDA, "staging: %s", cudaGetErrorString(e));
    }
    uint8_t *h = static_cast<uint8_t *>(slot->host);
    size_t off = 0;
    auto put = [&](const void *src, size_t n) {
      if (n) std::memcpy(h + off, src, n);
      const size_t o = off;
      off += align256(std::max<size_t>(n, 4));
      return dws + o;
    };
    const TileItem *d_tile = reinterpret_cast<const TileItem *>(put(pb.tile.data(), tile_inline ? 0 : sizeof(TileItem) * pb.tile.size()));
    if (!tile_inline) pl->tiles.ptr = d_tile;
    pl->p.row_list = reinterpret_cast<const int32_t *>(put(pb.row_list.data(), 4 * pb.row_list.size()));
    if (!dec_inline) {
      pl->dec.ptr = reinterpret_cast<const DecodeReq *>(put(pb.dec.data(), sizeof(DecodeReq) * pb.dec.size()));
      pl->dec.pre_ptr = reinterpret_cast<const int32_t *>(put(pb.dec_pre.data(), 4 * pb.dec_pre.size()));
    }
    if (!mrg_inline) {
      pl->mrg.ptr = reinterpret_cast<const MergeReq *>(put(pb.mrg.data(), sizeof(MergeReq) * pb.mrg.size()));
      pl->mrg.pre_ptr = reinterpret_cast<const int32_t *>(put(pb.mrg_pre.data(), 4 * pb.mrg_pre.size()));
    }
    if (has_fold) {  // the fold list, zeroed completion counters, the reduced merge list if large
      pl->p.fold = reinterpret_cast<const FoldReq *>(put(pb.fold.data(), sizeof(FoldReq) * pb.fold.size()));
      const std::vector<uint32_t> zeros(2 * (size_t)pb.n_casc_items, 0u);
      pl->p.fold_flags = reinterpret_cast<unsigned *>(put(zeros.data(), 4 * zeros.size()));
      if (!mrg_red_inline) {
        pl->mrg_red.ptr = reinterpret_cast<const MergeReq *>(put(pb.mrg_red.data(), sizeof(MergeReq) * pb.mrg_red.size()));
        pl->mrg_red.pre_ptr = reinterpret_cast<const int32_t *>(put(pb.mrg_red_pre.data(), 4 * pb.mrg_red_pre.size()));
      }
      pl->has_fold = true;
    }
    // upload on the side stream, ordered after everything already enqueued on `stream`
    // (WAR on the workspace), so the decode launch on `stream` does not queue behind a
    // copy-engine transfer
    pl->ev_up0 = p->ev_up0;
    pl->ev_up1 = p->ev_up1;
    e = cudaEventRecord(pl->ev_up0, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->aux, pl->ev_up0, 0);
    if (e == cudaSuccess) e = p->staging.upload(slot, ws, off, p->aux);
    if (e == cudaSuccess) e = cudaEventRecord(pl->ev_up1, p->aux);
    if (e != cudaSuccess) {
      delete pl;
      return fail(KVA_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
    }
    pl->uploaded = true;
  }
  hs.lap("plan.upload");
  pl->aux = p->aux;
  pl->pool = p;
  pl->ev_fork = p->ev_fork;
  pl->ev_join = p->ev_join;
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->desc.device);
    const int64_t tc_opt = opt(kOptTileCtas);
    pl->overlap = opt(kOptOverlap) != 0;
    // standalone time estimates from measured rates: ~3.9 TFLOP/s per SM for
    // the tcgen05 tile kernel, 6.7 TB/s for the decode stream
    const double t_tile = (double)pb.tile_flops / (nsm * 3.9e12);
    const double t_dec = (double)pb.stats.decode_kv_bytes / 6.7e12;
    if (tc_opt > 0) {
      pl->tile_ctas = (int)std::min<int64_t>(tc_opt, nsm);
    } else if (pb.dec.empty() || pb.tile.empty() || !pl->overlap || t_tile > 1.5 * t_dec) {
      // tile-dominated batches (e.g. 8k chunks): run the tile kernel on every SM, then decode
      pl->overlap = false;
      pl->tile_ctas = nsm;
    } else {
      // split the SMs: proportional to the standalone times, skewed 1.5x towards the tile
      // kernel because the decode stream saturates HBM on ~94-104 SMs (profiles/r01b
      // decode_sm_curve.log: 6.8 TB/s on 104, 6.3 on 74); llama7b: 54 of 148 (step 403 us vs
      // 420 at 44 without the eviction selection co-running, equal with it); >= 1/4 each
      const double f = 1.5 * t_tile / (t_tile + t_dec);
      pl->tile_ctas = std::max(nsm / 4, std::min(nsm - nsm / 4, (int)(nsm * f + 0.5)));
    }
  }
  const auto t3 = std::chrono::steady_clock::now();
  hs.lap("plan.split");
  pl->stats.host_validate_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  pl->stats.host_build_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t2 - t1).count();
  pl->stats.host_total_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t3 - t0).count();
  pl->n_dec = pb.dec_pre.back() * b->num_kv_heads;
  pl->n_tile = (int)pb.tile.size();
  pl->n_mrows = pb.mrg_pre.back() * b->num_kv_heads;
  pl->n_mrows_red = pb.mrg_red_pre.back() * b->num_kv_heads;
  AttnParams &ap = pl->p;
  ap.k_pool = static_cast<const uint16_t *>(p->desc.k_pool);
  ap.v_pool = static_cast<const uint16_t *>(p->desc.v_pool);
  ap.num_blocks = p->desc.num_blocks;
  ap.Hkv = b->num_kv_heads;
  ap.Hq = b->num_q_heads;
  ap.g = b->num_q_heads / b->num_kv_heads;
  ap.d = b->head_dim;
  ap.block_table = b->block_table;
  ap.max_blocks = b->max_blocks;
  const double scale = b->sm_scale > 0 ? (double)b->sm_scale : 1.0 / std::sqrt((double)b->head_dim);
  ap.scale_log2 = (float)(scale * 1.4426950408889634);
  ap.part_o = reinterpret_cast<float *>(dws + arrays);
  ap.part_lse = reinterpret_cast<float *>(dws + arrays + align256((size_t)pb.n_slots * b->head_dim * 4));
  *out = pl;
  return KVA_OK;
}

extern "C" kva_status hybrid_attention_plan(kva_pool *p, const kva_batch_desc *b, void *ws,
                                            size_t ws_bytes, kva_stream_t stream, kva_plan **out) {
  return plan_impl(p, b, ws, ws_bytes, stream, out, false);
}

extern "C" kva_status kv_append_plan(kva_pool *p, kva_batch_desc *b, const void *k_new, const void *v_new,
                                     int64_t stride_tok, int32_t *deficit, void *ws_append, size_t ws_append_bytes,
                                     void *ws_attn, size_t ws_attn_bytes, kva_stream_t stream, kva_plan **out) {
  if (!out) return fail(KVA_ERR_INVALID, "null plan pointer");
  *out = nullptr;
  if (deficit) *deficit = 0;
  // one validation (the append's: the resident part; the plan reads no block id, and the
  // append itself writes every new position's entry), then the plan — so a plan error leaves
  // the pool untouched — then the append (its own errors: the plan is destroyed)
  HSection hs;
  kva_status st = validate_desc(p, b, 1);
  hs.lap("append_plan.validate");
  if (st != KVA_OK) return st;
  kva_plan *pl = nullptr;
  if ((st = plan_impl(p, b, ws_attn, ws_attn_bytes, stream, &pl, true)) != KVA_OK) return st;
  st = append_impl(p, b, k_new, v_new, stride_tok, deficit, ws_append, ws_append_bytes, stream, true);
  if (st != KVA_OK) {
    const std::string msg = g_err;  // kva_plan_destroy does not touch it; keep the append's message
    delete pl;
    g_err = msg;
    return st;
  }
  *out = pl;
  return KVA_OK;
}

extern "C" kva_status kva_plan_destroy(kva_plan *pl) {
  delete pl;
  return KVA_OK;
}

extern "C" kva_status kva_plan_get_stats(const kva_plan *pl, kva_plan_stats *st) {
  if (!pl || !st) return fail(KVA_ERR_INVALID, "null argument");
  *st = pl->stats;
  return KVA_OK;
}

extern "C" kva_status hybrid_attention_run_phases(const kva_plan *pl, const void *q, int64_t q_st,
                                                  int64_t q_sh, void *out, int64_t o_st,
                                                  int64_t o_sh, int32_t out_dtype, float *lse,
                                                  int32_t phases, kva_stream_t stream) {
  if (!pl) return fail(KVA_ERR_INVALID, "null plan");
  if (pl->n_dec + pl->n_tile == 0) return KVA_OK;
  if (!q || !out) return fail(KVA_ERR_INVALID, "q and out are required");
  if (out_dtype != KVA_OUT_BF16 && out_dtype != KVA_OUT_F32)
    return fail(KVA_ERR_INVALID, "out_dtype must be KVA_OUT_BF16 or KVA_OUT_F32");
  if ((reinterpret_cast<uintptr_t>(q) & 3) || (q_st & 1) || (q_sh & 1))
    return fail(KVA_ERR_INVALID, "q must be 4-byte aligned with even strides");
  const int vec = out_dtype == KVA_OUT_F32 ? 16 : 8;
  if ((reinterpret_cast<uintptr_t>(out) & (vec - 1)) || (o_st % 4) || (o_sh % 4))
    return fail(KVA_ERR_INVALID, "out must be %d-byte aligned with strides %% 4 == 0", vec);
  HSection hs;
  DeviceGuard dg(pl->device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  AttnParams p = pl->p;
  p.q = static_cast<const uint16_t *>(q);
  p.q_stride_tok = q_st;
  p.q_stride_head = q_sh;
  p.out = out;
  p.o_stride_tok = o_st;
  p.o_stride_head = o_sh;
  p.out_f32 = out_dtype == KVA_OUT_F32;
  p.lse = lse;
  p.dbg = nullptr;
  p.span = pl->span;
  p.n_out_extra = pl->n_out_extra;
  for (int i = 0; i < kMaxOutExtra; ++i) p.out_extra[i] = pl->out_extra[i];
  p.debug_flags = (int32_t)opt(kOptDebugFlags);
  if (const int64_t ts_addr = opt(kOptDebugTs)) p.dbg = reinterpret_cast<unsigned long long *>(ts_addr);
  const bool do_tile = (phases & KVA_PHASE_TILE) && pl->n_tile > 0;
  const bool do_dec = (phases & KVA_PHASE_DECODE) && pl->n_dec > 0;
  const bool fork = do_tile && do_dec && pl->overlap;
  const bool pdl_mode = opt(kOptPdl) != 0;
  // the plan's fold (decode-epilogue merge of cascade members) needs the tile kernel resident
  // before the decode kernel: only in the one-stream PDL mode with both kernels in this run
  // (and the merge in the same run: it then uses the list without the folded requests)
  const bool fold = fork && pdl_mode && pl->has_fold && (phases & KVA_PHASE_MERGE) && opt(kOptFold) != 0;
  if (do_tile) ++pl->runs;  // the epoch the tile kernel's fold counters reach in this run
  p.epoch = pl->runs;
  p.fold_on = fold ? 1 : 0;
  cudaStream_t ts = s;
  if (fork && !pdl_mode) {  // tile kernel first on the high-priority side stream, then decode on `s`
    CUDA_TRY(cudaEventRecord(pl->ev_fork, s));
    CUDA_TRY(cudaStreamWaitEvent(pl->aux, pl->ev_fork, 0));
    ts = pl->aux;
  }
  // kernels reading uploaded plan arrays on `s` wait for the side-stream upload (the tile
  // kernel on the side stream is ordered after it already)
  auto wait_upload = [&](bool needed) -> kva_status {
    if (needed && pl->uploaded) CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_up1, 0));
    return KVA_OK;
  };
  // rows appended on the side stream are read only by the tile kernel: on `s` it waits for them
  // (on the side stream it is ordered after them already)
  auto wait_append = [&]() -> kva_status {
    return KVA_OK;
  };
  auto run_tile = [&]() -> kva_status {
    if (ts == s && wait_upload(true) != KVA_OK) return KVA_ERR_CUDA;
    if (ts == s && wait_append() != KVA_OK) return KVA_ERR_CUDA;
    if (pl->t_ev[0]) CUDA_TRY(cudaEventRecord(pl->t_ev[0], ts));
    CUDA_TRY(launch_tile_tc2(p, &pl->tmk, &pl->tmv, pl->tiles, fork ? pl->tile_ctas : 0, ts,
                             pl->has3d ? &pl->tmv3 : nullptr, pl->has3d ? &pl->tmk4 : nullptr));
    if (pl->t_ev[1]) CUDA_TRY(cudaEventRecord(pl->t_ev[1], ts));
    return KVA_OK;
  };
  auto run_decode = [&]() -> kva_status {
    if (wait_upload(pl->dec.ptr != nullptr) != KVA_OK) return KVA_ERR_CUDA;
    // overlapped: the decode kernel also waits for the side-stream append, so it does not
    // become ready before the tile kernel (launched first, high priority) and fill every SM
    if (fork && wait_append() != KVA_OK) return KVA_ERR_CUDA;
    if (pl->t_ev[2]) CUDA_TRY(cudaEventRecord(pl->t_ev[2], s));
    CUDA_TRY(launch_decode(p, &pl->tmk, &pl->tmv, pl->dec, pl->n_dec, s, false, pl->has3d ? &pl->tmk3 : nullptr,
                           pl->has3d ? &pl->tmv3 : nullptr));
    if (pl->t_ev[3]) CUDA_TRY(cudaEventRecord(pl->t_ev[3], s));
    return KVA_OK;
  };
  // overlapped, PDL mode (default for the tcgen05 tile kernel + decode v2): both kernels on
  // `s`; the persistent tile kernel launches first and, once all its CTAs are resident, lets
  // the decode kernel (programmatic dependent launch) start on the remaining SMs.  This fixes
  // the SM split: with two streams the decode kernel's 2-CTA/SM grid could be dispatched first
  // and hold every SM until its first wave retired.  Timing events bracket the pair.
  if (fork && pdl_mode) {
    if (wait_upload(true) != KVA_OK || wait_append() != KVA_OK) return KVA_ERR_CUDA;
    if (pl->t_ev[0]) CUDA_TRY(cudaEventRecord(pl->t_ev[0], s));
    if (pl->t_ev[2]) CUDA_TRY(cudaEventRecord(pl->t_ev[2], s));
    hs.lap("run.prep");
    CUDA_TRY(launch_tile_tc2(p, &pl->tmk, &pl->tmv, pl->tiles, pl->tile_ctas, s, pl->has3d ? &pl->tmv3 : nullptr,
                             pl->has3d ? &pl->tmk4 : nullptr));
    hs.lap("run.launch_tile");
    CUDA_TRY(launch_decode(p, &pl->tmk, &pl->tmv, pl->dec, pl->n_dec, s, /*pdl=*/true,
                           pl->has3d ? &pl->tmk3 : nullptr, pl->has3d ? &pl->tmv3 : nullptr));
    hs.lap("run.launch_decode");
    if (pl->t_ev[1]) CUDA_TRY(cudaEventRecord(pl->t_ev[1], s));
    if (pl->t_ev[3]) CUDA_TRY(cudaEventRecord(pl->t_ev[3], s));
    const ReqList<MergeReq> &mrg = fold ? pl->mrg_red : pl->mrg;
    const int n_mrows = fold ? pl->n_mrows_red : pl->n_mrows;
    if ((phases & KVA_PHASE_MERGE) && n_mrows > 0) CUDA_TRY(launch_merge(p, mrg, n_mrows, s));
    // the decode kernel does not wait for the tile kernel: when it is the last kernel of the
    // run, a join kernel ends it, so the completion of the run's last kernel implies the tile
    // kernel's (the next kv_truncate / kv_append are programmatic dependents that wait only
    // for their immediate predecessor)
    else if (do_dec) CUDA_TRY(launch_join(s));
    hs.lap("run.launch_merge");
    return KVA_OK;
  }
  // sequential mode: decode first (its CTAs share SMs with a concurrently running eviction
  // selection on another stream), then the tile kernel on every SM
  kva_status rs = KVA_OK;
  if (fork) {
    if (do_tile && (rs = run_tile()) != KVA_OK) return rs;
    if (do_dec && (rs = run_decode()) != KVA_OK) return rs;
  } else {
    if (do_dec && (rs = run_decode()) != KVA_OK) return rs;
    if (do_tile && (rs = run_tile()) != KVA_OK) return rs;
  }
  if (fork) {
    CUDA_TRY(cudaEventRecord(pl->ev_join, pl->aux));
    CUDA_TRY(cudaStreamWaitEvent(s, pl->ev_join, 0));
  }
  if ((phases & KVA_PHASE_MERGE) && pl->n_mrows > 0) {
    if (wait_upload(pl->mrg.ptr != nullptr) != KVA_OK) return KVA_ERR_CUDA;
    CUDA_TRY(launch_merge(p, pl->mrg, pl->n_mrows, s));
  }
  // a full run leaves `s` ordered after every side-stream write of this step
  if ((phases & KVA_PHASE_ALL) == KVA_PHASE_ALL && wait_append() != KVA_OK) return KVA_ERR_CUDA;
  return KVA_OK;
}

extern "C" kva_status hybrid_attention_run(const kva_plan *pl, const void *q, int64_t q_st,
                                           int64_t q_sh, void *out, int64_t o_st, int64_t o_sh,
                                           int32_t out_dtype, float *lse, kva_stream_t stream) {
  return hybrid_attention_run_phases(pl, q, q_st, q_sh, out, o_st, o_sh, out_dtype, lse,
                                     KVA_PHASE_ALL, stream);
}

extern "C" kva_status kva_plan_set_outputs(kva_plan *pl, int32_t n, void *const *outs) {
  if (!pl || n < 0 || n > kMaxOutExtra || (n > 0 && !outs))
    return fail(KVA_ERR_INVALID, "n must be in [0, %d] with a pointer array", kMaxOutExtra);
  for (int i = 0; i < n; ++i)
    if (!outs[i] || (reinterpret_cast<uintptr_t>(outs[i]) & 15))
      return fail(KVA_ERR_INVALID, "extra output %d is null or not 16-byte aligned", i);
  pl->n_out_extra = n;
  for (int i = 0; i < kMaxOutExtra; ++i) pl->out_extra[i] = i < n ? outs[i] : nullptr;
  return KVA_OK;
}

extern "C" kva_status kva_plan_set_span_buffer(kva_plan *pl, unsigned long long *dev_span) {
  if (!pl) return fail(KVA_ERR_INVALID, "null plan");
  pl->span = dev_span;
  return KVA_OK;
}

extern "C" kva_status kva_plan_set_timing_events(kva_plan *pl, void *tile_begin, void *tile_end,
                                                 void *decode_begin, void *decode_end) {
  if (!pl) return fail(KVA_ERR_INVALID, "null plan");
  pl->t_ev[0] = static_cast<cudaEvent_t>(tile_begin);
  pl->t_ev[1] = static_cast<cudaEvent_t>(tile_end);
  pl->t_ev[2] = static_cast<cudaEvent_t>(decode_begin);
  pl->t_ev[3] = static_cast<cudaEvent_t>(decode_end);
  return KVA_OK;
}

extern "C" kva_status kva_plan_launch_count(const kva_plan *pl, int32_t phases, int32_t *n) {
  if (!pl || !n) return fail(KVA_ERR_INVALID, "null argument");
  const bool tile = (phases & KVA_PHASE_TILE) && pl->n_tile > 0, dec = (phases & KVA_PHASE_DECODE) && pl->n_dec > 0;
  const bool pdl_fork = tile && dec && pl->overlap && opt(kOptPdl) != 0;
  const bool fold = pdl_fork && pl->has_fold && (phases & KVA_PHASE_MERGE) && opt(kOptFold) != 0;
  const bool merge = (phases & KVA_PHASE_MERGE) && (fold ? pl->n_mrows_red : pl->n_mrows) > 0;
  // + the join kernel that ends an overlapped PDL run without a merge (hybrid_attention_run)
  const bool join = pdl_fork && !merge;
  *n = tile + dec + merge + join;
  return KVA_OK;
}

// ------------------------------------------------------------------------------------------
// block release (recompute-mode preemption / finished requests)
// ------------------------------------------------------------------------------------------
// Marks ids[0, n) allocated -> free in the host mirror; on an invalid list (out of range,
// already free, listed twice) every mark is undone and the error returned.
static kva_status mark_released(kva_pool *p, const int32_t *ids, int64_t n) {
  const int nb = p->desc.num_blocks;
  for (int64_t i = 0; i < n; ++i) {
    const int32_t id = ids[i];
    kva_status st = KVA_OK;
    if (id < 0 || id >= nb) st = fail(KVA_ERR_INVALID, "block id %d out of range", id);
    else if ((p->free_host[id >> 5] >> (id & 31)) & 1u) {
      bool twice = false;  // set by this call (an earlier element) or free before it?
      for (int64_t j = 0; j < i && !twice; ++j) twice = ids[j] == id;
      st = twice ? fail(KVA_ERR_INVALID, "block %d listed twice", id) : fail(KVA_ERR_INVALID, "block %d is already free", id);
    }
    if (st != KVA_OK) {
      for (int64_t j = 0; j < i; ++j) p->free_host[ids[j] >> 5] &= ~(1u << (ids[j] & 31));
      return st;
    }
    p->free_host[id >> 5] |= 1u << (id & 31);
  }
  p->n_free += n;
  return KVA_OK;
}

extern "C" kva_status kv_release_blocks(kva_pool *p, const int32_t *ids, int64_t n,
                                        kva_stream_t stream) {
  if (!p || n < 0 || (n > 0 && !ids)) return fail(KVA_ERR_INVALID, "bad arguments");
  if (n == 0) return KVA_OK;
  HSection hs;
  kva_status st = mark_released(p, ids, n);
  hs.lap("release.check");
  if (st != KVA_OK) return st;
  DeviceGuard dg(p->desc.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // ids travel as kernel parameters (<= kReleaseBatch per launch): no device scratch,
  // no host<->device copy, stream-ordered like every other call
  for (int64_t off = 0; off < n; off += kReleaseBatch) {
    const int cnt = (int)std::min<int64_t>(kReleaseBatch, n - off);
    CUDA_TRY(launch_release_ids(p->desc.free_bits, ids + off, cnt, s));
  }
  hs.lap("release.launch");
  return KVA_OK;
}

extern "C" kva_status kv_truncate(kva_pool *p, kva_batch_desc *b, const int32_t *keep_len, kva_stream_t stream) {
  if (!p || !b || (b->num_reqs > 0 && !keep_len)) return fail(KVA_ERR_INVALID, "bad arguments");
  if (b->num_reqs < 0) return fail(KVA_ERR_INVALID, "num_reqs < 0");
  if (b->num_reqs == 0) return KVA_OK;
  if (!b->ctx_len || !b->block_table || !b->block_table_host || b->max_blocks <= 0)
    return fail(KVA_ERR_INVALID, "ctx_len, block_table, block_table_host and max_blocks required");
  HSection hs;
  std::vector<int32_t> tbl, ids;
  for (int i = 0; i < b->num_reqs; ++i) {
    const int keep = keep_len[i], ctx = b->ctx_len[i];
    if (keep == -1) continue;
    if (keep < 0 || keep > ctx || ctx > b->max_blocks * kBlock)
      return fail(KVA_ERR_INVALID, "request %d: keep_len %d not in [0, ctx_len %d]", i, keep, ctx);
    const int k0 = cdiv(keep, kBlock);
    if (b->group_of && b->group_of[i] >= 0 && b->group_prefix_blocks && b->group_of[i] < b->num_groups &&
        k0 < b->group_prefix_blocks[b->group_of[i]])
      return fail(KVA_ERR_GROUP, "request %d: truncation inside its shared prefix", i);
    const int32_t *row = b->block_table_host + (int64_t)i * b->max_blocks;
    for (int k = k0; k < cdiv(ctx, kBlock); ++k) {
      if (row[k] == -1) continue;
      tbl.push_back(i * b->max_blocks + k);
      ids.push_back(row[k]);
    }
  }
  const int64_t n = (int64_t)ids.size();
  if (n == 0) return KVA_OK;
  kva_status st = mark_released(p, ids.data(), n);
  hs.lap("truncate.check");
  if (st != KVA_OK) return st;
  DeviceGuard dg(p->desc.device);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  for (int64_t off = 0; off < n; off += kReleaseBatch) {
    const int cnt = (int)std::min<int64_t>(kReleaseBatch, n - off);
    CUDA_TRY(launch_release_ids(p->desc.free_bits, ids.data() + off, cnt, s, tbl.data() + off, b->block_table));
  }
  for (int32_t t : tbl) b->block_table_host[t] = -1;
  hs.lap("truncate.launch");
  return KVA_OK;
}

extern "C" kva_status hybrid_attention(kva_pool *p, const kva_batch_desc *b, const void *q,
                                       int64_t q_st, int64_t q_sh, void *out, int64_t o_st,
                                       int64_t o_sh, int32_t out_dtype, float *lse, void *ws,
                                       size_t ws_bytes, kva_stream_t stream) {
  kva_plan *pl = nullptr;
  kva_status st = hybrid_attention_plan(p, b, ws, ws_bytes, stream, &pl);
  if (st != KVA_OK) return st;
  st = hybrid_attention_run(pl, q, q_st, q_sh, out, o_st, o_sh, out_dtype, lse, stream);
  kva_plan_destroy(pl);
  return st;
}

// ------------------------------------------------------------------------------------------
// burst-reserve threshold + KV-manager step
// ------------------------------------------------------------------------------------------
extern "C" kva_status kv_pool_set_threshold(kva_pool *p, int64_t threshold_blocks) {
  if (!p) return fail(KVA_ERR_INVALID, "null pool");
  if (threshold_blocks > p->desc.num_blocks)
    return fail(KVA_ERR_INVALID, "threshold %lld > num_blocks %d", (long long)threshold_blocks, p->desc.num_blocks);
  p->threshold_blocks = threshold_blocks < 0 ? -1 : threshold_blocks;
  return KVA_OK;
}

extern "C" kva_status kv_pool_set_active_blocks(kva_pool *p, int64_t active_blocks) {
  if (!p) return fail(KVA_ERR_INVALID, "null pool");
  if (active_blocks < 0 || active_blocks > p->desc.num_blocks)
    return fail(KVA_ERR_INVALID, "active_blocks %lld out of [0, num_blocks]", (long long)active_blocks);
  p->active_blocks = active_blocks;
  return KVA_OK;
}

namespace {
std::mutex g_mgr_mu;
Staging g_mgr_staging;  // pinned upload ring of the manager step (process-wide, mutex-guarded)

kva_status manager_validate(const kva_block_meta *m, const kva_manager_update *u, int64_t *tot_out) {
  if (!m || !u) return fail(KVA_ERR_INVALID, "null argument");
  const int64_t n = m->num_blocks;
  *tot_out = 0;
  if (n < 0 || n > INT32_MAX) return fail(KVA_ERR_INVALID, "num_blocks out of range");
  if (n > 0 && (!m->state || !m->rc || !m->lat)) return fail(KVA_ERR_INVALID, "state, rc, lat required");
  if (u->n_chains < 0 || u->pool_len < 0 || u->del_len < 0) return fail(KVA_ERR_INVALID, "negative counts");
  if (u->pool_len > 0 && !u->pool_ids) return fail(KVA_ERR_INVALID, "pool_ids required");
  if (u->del_len > 0 && (!u->del_ids || u->recount)) return fail(KVA_ERR_INVALID, "del_ids only in incremental mode");
  if (u->n_chains > 0 && u->chains_on_device) {
    if (!u->chain_indptr || !u->chain_state || (u->n_chain_ids > 0 && !u->chain_ids))
      return fail(KVA_ERR_INVALID, "chain arrays required");
    if (u->n_chain_ids < 0 || u->n_chain_ids > INT32_MAX) return fail(KVA_ERR_INVALID, "n_chain_ids out of range");
    *tot_out = u->n_chain_ids;
  } else if (u->n_chains > 0) {
    if (!u->chain_indptr || !u->chain_state) return fail(KVA_ERR_INVALID, "chain arrays required");
    if (u->chain_indptr[0] != 0) return fail(KVA_ERR_INVALID, "chain_indptr[0] != 0");
    for (int32_t j = 0; j < u->n_chains; ++j) {
      if (u->chain_indptr[j + 1] < u->chain_indptr[j]) return fail(KVA_ERR_INVALID, "chain_indptr not monotone");
      if (u->chain_state[j] > KVA_BLK_FINISHED_OFFLINE) return fail(KVA_ERR_INVALID, "chain %d: bad state", j);
    }
    const int64_t tot = u->chain_indptr[u->n_chains];
    if (tot > 0 && !u->chain_ids) return fail(KVA_ERR_INVALID, "chain_ids required");
    const int32_t *cid = u->chain_ids;
    uint32_t bad = 0;
    for (int64_t e = 0; e < tot; ++e) bad |= (uint32_t)cid[e] >= (uint32_t)n;  // vectorised
    if (bad) return fail(KVA_ERR_INVALID, "chain id out of range");
    *tot_out = tot;
  }
  return KVA_OK;
}

size_t manager_ws_bytes(int64_t n, int64_t tot, int32_t nc) {
  return align256((size_t)tot * 4) + align256((size_t)(nc + 1) * 4) + align256((size_t)nc + 1) +
         (tot > 0 ? align256((size_t)n * 4) : 0) + 256;
}
}  // namespace

extern "C" kva_status kv_manager_step_workspace_size(const kva_block_meta *m, const kva_manager_update *u,
                                                     size_t *bytes) {
  if (!m || !u || !bytes) return fail(KVA_ERR_INVALID, "null argument");
  const int64_t tot = u->n_chains <= 0 ? 0
                      : u->chains_on_device ? std::max<int64_t>(0, u->n_chain_ids)
                      : (u->chain_indptr ? u->chain_indptr[u->n_chains] : 0);
  *bytes = manager_ws_bytes(m->num_blocks, tot, std::max(0, u->n_chains));
  return KVA_OK;
}

namespace {
struct MgrPrep {
  const int32_t *d_ids = nullptr, *d_ind = nullptr;
  const uint8_t *d_st = nullptr;
  int32_t *win = nullptr;
  int64_t tot = 0;
  int32_t nc = 0;
};
// validation + (host chains) the upload of the raw chains into the workspace
kva_status manager_prepare(const kva_block_meta *m, const kva_manager_update *u, uint64_t *keys, void *ws,
                           size_t ws_bytes, cudaStream_t s, MgrPrep &o) {
  int64_t tot = 0;
  HSection hs;
  kva_status st = manager_validate(m, u, &tot);
  hs.lap("manager.validate");
  if (st != KVA_OK) return st;
  if (m->num_blocks > 0 && !keys) return fail(KVA_ERR_INVALID, "keys_out required");
  const int32_t nc = tot > 0 ? u->n_chains : 0;
  const size_t need = manager_ws_bytes(m->num_blocks, tot, nc);
  if (tot > 0 && (!ws || ws_bytes < need))
    return fail(KVA_ERR_INVALID, "kv_manager_step workspace too small (%zu < %zu)", ws_bytes, need);
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(KVA_ERR_INVALID, "workspace must be 256-B aligned");
  uint8_t *w = static_cast<uint8_t *>(ws);
  const size_t o_ind = align256((size_t)tot * 4), o_st = o_ind + align256((size_t)(nc + 1) * 4);
  const size_t o_win = o_st + align256((size_t)nc + 1);
  o.d_ids = reinterpret_cast<const int32_t *>(w);
  o.d_ind = reinterpret_cast<const int32_t *>(w + o_ind);
  o.d_st = w + o_st;
  o.win = reinterpret_cast<int32_t *>(w + o_win);
  o.tot = tot;
  o.nc = nc;
  if (u->chains_on_device) {
    o.d_ids = u->chain_ids;
    o.d_ind = u->chain_indptr;
    o.d_st = u->chain_state;
  } else if (tot > 0) {  // upload the raw chains (no per-element host work beyond validation)
    std::lock_guard<std::mutex> lk(g_mgr_mu);
    Staging::Slot *slot = nullptr;
    CUDA_TRY(g_mgr_staging.get(o_win, &slot));
    uint8_t *h = static_cast<uint8_t *>(slot->host);
    std::memcpy(h, u->chain_ids, (size_t)tot * 4);
    std::memcpy(h + o_ind, u->chain_indptr, (size_t)(nc + 1) * 4);
    std::memcpy(h + o_st, u->chain_state, (size_t)nc);
    CUDA_TRY(g_mgr_staging.upload(slot, ws, o_st + nc, s));
  }
  hs.lap("manager.upload");
  return KVA_OK;
}
}  // namespace

extern "C" kva_status kv_manager_step(const kva_block_meta *m, const kva_manager_update *u, uint64_t *keys,
                                      int64_t *n_active, void *ws, size_t ws_bytes, kva_stream_t stream) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  MgrPrep o;
  if (kva_status st = manager_prepare(m, u, keys, ws, ws_bytes, s, o); st != KVA_OK) return st;
  HSection hs;
  CUDA_TRY(launch_manager_step(m->state, m->rc, m->lat, m->depth, m->num_blocks, u->now, o.d_ids, o.tot, o.d_ind,
                               o.d_st, o.nc, o.win, u->recount != 0, u->pool_ids, u->pool_len, u->del_ids,
                               u->del_len, keys, n_active, s));
  hs.lap("manager.launch");
  return KVA_OK;
}

extern "C" kva_status kv_manager_step_select(const kva_block_meta *m, const kva_manager_update *u, uint64_t *keys,
                                             int64_t *n_active, void *ws, size_t ws_bytes, int64_t k,
                                             int32_t *out_ids, void *sel_ws, size_t sel_ws_bytes,
                                             kva_stream_t stream) {
  if (!m) return fail(KVA_ERR_INVALID, "null argument");
  const int64_t n = m->num_blocks;
  if (k < 0) return fail(KVA_ERR_INVALID, "k must be >= 0");
  if (n >= (1ll << 31)) return fail(KVA_ERR_UNSUPPORTED, "n >= 2^31");
  if (k > 0 && n > 0 && !out_ids) return fail(KVA_ERR_INVALID, "out_ids required");
  const size_t need = evict_select_ws_bytes(n, k) + 256;
  if (!sel_ws || sel_ws_bytes < need)
    return fail(KVA_ERR_INVALID, "selection workspace too small (%zu < %zu)", sel_ws_bytes, need);
  if (k == 0 || n == 0)  // nothing to select: the manager step alone
    return kv_manager_step(m, u, keys, n_active, ws, ws_bytes, stream);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  MgrPrep o;
  if (kva_status st = manager_prepare(m, u, keys, ws, ws_bytes, s, o); st != KVA_OK) return st;
  HSection hs;
  MgrArgs ma = make_mgr_args(m->state, m->rc, m->lat, m->depth, n, u->now, o.d_ids, o.tot, o.d_ind, o.d_st, o.nc,
                             o.win, u->recount != 0, u->pool_ids, u->pool_len, u->del_ids, u->del_len, keys,
                             n_active);
  uint8_t *w = static_cast<uint8_t *>(sel_ws);
  CUDA_TRY(launch_evict_select(keys, n, k, out_ids, reinterpret_cast<int64_t *>(w), nullptr, w + 256,
                               sel_ws_bytes - 256, (int)opt(kOptEvictCtas), s, &ma));
  hs.lap("manager.launch");
  return KVA_OK;
}

// ------------------------------------------------------------------------------------------
// eviction (a8)
// ------------------------------------------------------------------------------------------
extern "C" kva_status evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                                 const uint16_t *depth, int64_t n, uint64_t *keys,
                                 kva_stream_t stream) {
  if (n < 0) return fail(KVA_ERR_INVALID, "n < 0");
  if (n == 0) return KVA_OK;
  if (!state || !rc || !lat || !keys) return fail(KVA_ERR_INVALID, "state, rc, lat, keys required");
  CUDA_TRY(launch_evict_keys(state, rc, lat, depth, n, keys, reinterpret_cast<cudaStream_t>(stream)));
  return KVA_OK;
}

extern "C" kva_status evict_select_workspace_size(int64_t n, int64_t k, size_t *bytes) {
  if (!bytes || n < 0 || k < 0) return fail(KVA_ERR_INVALID, "bad arguments");
  *bytes = evict_select_ws_bytes(n, k) + 256;
  return KVA_OK;
}

extern "C" kva_status evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                                   int64_t *n_selected, int32_t apply, kva_pool *pool, void *ws,
                                   size_t ws_bytes, kva_stream_t stream) {
  if (n < 0 || k < 0) return fail(KVA_ERR_INVALID, "n and k must be >= 0");
  if (n >= (1ll << 31)) return fail(KVA_ERR_UNSUPPORTED, "n >= 2^31");
  if (apply && !n_selected) return fail(KVA_ERR_INVALID, "apply requires n_selected");
  if (n_selected) *n_selected = 0;
  if (apply && !pool) return fail(KVA_ERR_INVALID, "apply requires the pool");
  if (apply && pool && n > pool->desc.num_blocks) return fail(KVA_ERR_INVALID, "n > pool blocks");
  if (k == 0 || n == 0) return k == 0 ? KVA_OK : fail(KVA_EVICTION_SHORT, "no evictable blocks");
  if (!keys || !out_ids) return fail(KVA_ERR_INVALID, "keys and out_ids required");
  const size_t need = evict_select_ws_bytes(n, k) + 256;
  if (!ws || ws_bytes < need) return fail(KVA_ERR_INVALID, "evict_select workspace too small (%zu < %zu)", ws_bytes, need);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t *w = static_cast<uint8_t *>(ws);
  int64_t *d_count = reinterpret_cast<int64_t *>(w);
  const int ctas = (int)opt(kOptEvictCtas);
  CUDA_TRY(launch_evict_select(keys, n, k, out_ids, d_count, apply ? pool->desc.free_bits : nullptr, w + 256,
                               ws_bytes - 256, ctas, s));
  if (!n_selected) return KVA_OK;  // asynchronous mode: count stays on the device
  int64_t cnt = 0;
  CUDA_TRY(cudaMemcpyAsync(&cnt, d_count, sizeof cnt, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  *n_selected = cnt;
  if (apply && cnt > 0) {
    std::vector<int32_t> ids(cnt);
    CUDA_TRY(cudaMemcpy(ids.data(), out_ids, cnt * 4, cudaMemcpyDeviceToHost));
    for (int32_t id : ids) {
      uint32_t &wd = pool->free_host[id >> 5];
      if (!((wd >> (id & 31)) & 1u)) {
        wd |= 1u << (id & 31);
        pool->n_free++;
      }
    }
  }
  if (cnt < k) return fail(KVA_EVICTION_SHORT, "only %lld of %lld blocks evictable", (long long)cnt, (long long)k);
  return KVA_OK;
}
