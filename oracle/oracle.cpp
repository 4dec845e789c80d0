/*
 * oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY (not part of the product path).
 *
 * A plain, slow, obviously-correct fp64 CPU oracle for the hot path of
 * arxiv 2504.03651 ("co-scheduling online and offline LLM tasks"):
 *   - paged causal attention of a mixed batch (online decodes + offline
 *     chunked prefills that share resident prefix blocks),
 *   - the KV append with deterministic block allocation,
 *   - the task-aware eviction key (priority, LAT) and the eviction order.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_2504_03651_b200/.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "reading #n" = DESIGN.md §3 (the reading of a silent/ambiguous passage).
 *
 * Built with: g++ -O2 -std=c++17 -shared -fPIC -pthread (NO -ffast-math).
 */
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

/* Status values of the boundary contract; restated here, not
 * included from the product header. */
constexpr int ST_OK = 0;
constexpr int ST_INVALID = 1;
constexpr int ST_NEEDS_EVICTION = 3;
constexpr int ST_CAPACITY = 4;
constexpr int ST_EVICTION_SHORT = 5;
constexpr int ST_GROUP = 6;

constexpr int BLOCK = 16; /* "fixed-sized blocks" P:328; size 16 = reading #5 */

/* bf16 bit pattern -> exact double (reading #12: inputs are bf16 bits). */
double bf16(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return static_cast<double>(f);
}

struct Batch {
  int32_t num_reqs, num_q_heads, num_kv_heads, head_dim;
  const int32_t *q_indptr;           /* [R+1] */
  const int32_t *ctx_len;            /* [R]   */
  const int32_t *block_table;        /* [R][max_blocks] */
  int32_t max_blocks;
  const int32_t *group_of;           /* [R], -1 = none (may be null) */
  int32_t num_groups;
  const int32_t *group_prefix_blocks;/* [num_groups] */
  int32_t num_blocks;
  double sm_scale;                   /* <= 0 -> 1/sqrt(d) (reading #1) */
};

int q_len_of(const Batch &b, int i) { return b.q_indptr[i + 1] - b.q_indptr[i]; }

/* Structural checks shared by attention and append ("its tokens can be
 * scheduled only if the corresponding KV cache before the tokens are in the
 * memory"; group precondition = reading #8). */
int validate(const Batch &b, bool need_full_table) {
  if (b.num_reqs < 0 || b.num_q_heads <= 0 || b.num_kv_heads <= 0) return ST_INVALID;
  if (b.num_q_heads % b.num_kv_heads != 0) return ST_INVALID;
  if (b.q_indptr[0] != 0) return ST_INVALID;
  for (int i = 0; i < b.num_reqs; ++i) {
    int ql = q_len_of(b, i), ctx = b.ctx_len[i];
    if (ql < 1 || ql > ctx) return ST_INVALID;
    if (ctx > b.max_blocks * BLOCK) return ST_INVALID;
    if (need_full_table) {
      for (int blk = 0; blk < (ctx + BLOCK - 1) / BLOCK; ++blk) {
        int id = b.block_table[(int64_t)i * b.max_blocks + blk];
        if (id < 0 || id >= b.num_blocks) return ST_INVALID;
      }
    }
  }
  for (int i = 0; i < b.num_reqs; ++i) {
    int g = b.group_of ? b.group_of[i] : -1;
    if (g < 0) continue;
    if (g >= b.num_groups) return ST_GROUP;
    int np = b.group_prefix_blocks[g];
    if (np < 0) return ST_GROUP;
    /* every member's queries lie after the prefix */
    if (b.ctx_len[i] - q_len_of(b, i) < np * BLOCK) return ST_GROUP;
    /* its first n_pi table entries are the group's blocks (those of the first
     * member, in descriptor order) */
    int first = -1;
    for (int j = 0; j < b.num_reqs; ++j)
      if (b.group_of[j] == g) { first = j; break; }
    for (int blk = 0; blk < np; ++blk) {
      int a = b.block_table[(int64_t)i * b.max_blocks + blk];
      int c = b.block_table[(int64_t)first * b.max_blocks + blk];
      if (a != c || a < 0 || a >= b.num_blocks) return ST_GROUP;
    }
  }
  return ST_OK;
}

/* One output row by the plain definition of causal scaled-dot-product
 * attention over the paged cache (P:73-77 prefill/decode; P:82 chunked
 * prefill; P:328 paged blocks).  Query at absolute position p sees keys
 * [0, p] (readings #2-#4); q-head h reads kv-head floor(h/g) (reading #9);
 * plain softmax with natural-log lse (reading #10). */
void attend_row(const Batch &b, const uint16_t *kp, const uint16_t *vp,
                const uint16_t *q, int req, int j, int h, double *out, double *lse) {
  const int d = b.head_dim, Hq = b.num_q_heads, Hkv = b.num_kv_heads;
  const int g = Hq / Hkv, kvh = h / g;
  const int ql = q_len_of(b, req), ctx = b.ctx_len[req];
  const int p = ctx - ql + j;
  const int64_t row = b.q_indptr[req] + j;
  const double s = b.sm_scale > 0 ? b.sm_scale : 1.0 / std::sqrt((double)d);
  std::vector<double> qv(d), x(p + 1);
  for (int c = 0; c < d; ++c) qv[c] = bf16(q[(row * Hq + h) * d + c]);
  for (int t = 0; t <= p; ++t) {
    int blk = b.block_table[(int64_t)req * b.max_blocks + t / BLOCK];
    const uint16_t *kr = kp + (((int64_t)blk * Hkv + kvh) * BLOCK + t % BLOCK) * d;
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc += qv[c] * bf16(kr[c]);
    x[t] = s * acc;
  }
  double m = x[0];
  for (int t = 1; t <= p; ++t) m = std::max(m, x[t]);
  double Z = 0.0;
  std::vector<double> o(d, 0.0);
  for (int t = 0; t <= p; ++t) {
    double w = std::exp(x[t] - m);
    Z += w;
    int blk = b.block_table[(int64_t)req * b.max_blocks + t / BLOCK];
    const uint16_t *vr = vp + (((int64_t)blk * Hkv + kvh) * BLOCK + t % BLOCK) * d;
    for (int c = 0; c < d; ++c) o[c] += w * bf16(vr[c]);
  }
  for (int c = 0; c < d; ++c) out[c] = o[c] / Z;
  *lse = m + std::log(Z);
}

template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  nthreads = (int)std::min<int64_t>(nthreads, n);
  std::vector<std::thread> ts;
  for (int t = 0; t < nthreads; ++t)
    ts.emplace_back([&, t] {
      for (int64_t i = t; i < n; i += nthreads) f(i);
    });
  for (auto &t : ts) t.join();
}

Batch make_batch(int32_t num_reqs, int32_t Hq, int32_t Hkv, int32_t d,
                 const int32_t *q_indptr, const int32_t *ctx_len,
                 const int32_t *block_table, int32_t max_blocks,
                 const int32_t *group_of, int32_t num_groups,
                 const int32_t *group_prefix_blocks, int32_t num_blocks,
                 double sm_scale) {
  Batch b;
  b.num_reqs = num_reqs; b.num_q_heads = Hq; b.num_kv_heads = Hkv; b.head_dim = d;
  b.q_indptr = q_indptr; b.ctx_len = ctx_len; b.block_table = block_table;
  b.max_blocks = max_blocks; b.group_of = group_of; b.num_groups = num_groups;
  b.group_prefix_blocks = group_prefix_blocks; b.num_blocks = num_blocks;
  b.sm_scale = sm_scale;
  return b;
}

} // namespace

extern "C" {

/* Full attention: out [total_q][Hq][d] fp64, lse [total_q][Hq] fp64.
 * Group data is validated only; the result never depends on it (reading #7:
 * reuse replaces recomputation). */
int orc_attention(int32_t num_reqs, int32_t Hq, int32_t Hkv, int32_t d,
                  const int32_t *q_indptr, const int32_t *ctx_len,
                  const int32_t *block_table, int32_t max_blocks,
                  const int32_t *group_of, int32_t num_groups,
                  const int32_t *group_prefix_blocks, int32_t num_blocks,
                  double sm_scale, const uint16_t *k_pool, const uint16_t *v_pool,
                  const uint16_t *q, double *out, double *lse, int nthreads) {
  Batch b = make_batch(num_reqs, Hq, Hkv, d, q_indptr, ctx_len, block_table, max_blocks,
                       group_of, num_groups, group_prefix_blocks, num_blocks, sm_scale);
  int st = validate(b, true);
  if (st != ST_OK) return st;
  /* work unit = (request, q-head) */
  parallel_for((int64_t)num_reqs * Hq, nthreads, [&](int64_t u) {
    int i = (int)(u / Hq), h = (int)(u % Hq);
    for (int j = 0; j < q_len_of(b, i); ++j) {
      int64_t row = q_indptr[i] + j;
      attend_row(b, k_pool, v_pool, q, i, j, h, out + (row * Hq + h) * d, lse + row * Hq + h);
    }
  });
  return ST_OK;
}

/* Sampled rows: (q_row, head) pairs -> out [n][d], lse [n].  Rows are
 * independent, so each sampled row is exact (used at full sizes). */
int orc_attention_rows(int32_t num_reqs, int32_t Hq, int32_t Hkv, int32_t d,
                       const int32_t *q_indptr, const int32_t *ctx_len,
                       const int32_t *block_table, int32_t max_blocks,
                       const int32_t *group_of, int32_t num_groups,
                       const int32_t *group_prefix_blocks, int32_t num_blocks,
                       double sm_scale, const uint16_t *k_pool, const uint16_t *v_pool,
                       const uint16_t *q, const int32_t *rows, const int32_t *heads,
                       int64_t n, double *out, double *lse, int nthreads) {
  Batch b = make_batch(num_reqs, Hq, Hkv, d, q_indptr, ctx_len, block_table, max_blocks,
                       group_of, num_groups, group_prefix_blocks, num_blocks, sm_scale);
  int st = validate(b, true);
  if (st != ST_OK) return st;
  int total_q = q_indptr[num_reqs];
  for (int64_t s = 0; s < n; ++s)
    if (rows[s] < 0 || rows[s] >= total_q || heads[s] < 0 || heads[s] >= Hq) return ST_INVALID;
  parallel_for(n, nthreads, [&](int64_t s) {
    int row = rows[s];
    int i = (int)(std::upper_bound(q_indptr, q_indptr + num_reqs + 1, row) - q_indptr) - 1;
    attend_row(b, k_pool, v_pool, q, i, row - q_indptr[i], heads[s], out + s * d, lse + s);
  });
  return ST_OK;
}

/* KV append with deterministic allocation ("appending the corresponding
 * KV state to the cache"; capacity Eq.(5); readings #13, #14).
 * Requests in descriptor order, positions t in [ctx-q_len, ctx) ascending; if
 * table[i][t/16] == -1 the smallest free block id is taken.  The needed count
 * is computed first; if it exceeds the free blocks, NEEDS_EVICTION(deficit)
 * is returned and nothing changes ("on NeedsEviction, state
 * unchanged").  k_new/v_new: [total_q][Hkv][d]; free_bits: bit b of word
 * b/32 set = block b free. */
int orc_kv_append_t(int32_t num_reqs, int32_t Hkv, int32_t d,
                    const int32_t *q_indptr, const int32_t *ctx_len,
                    int32_t *block_table, int32_t max_blocks,
                    const int32_t *group_of, int32_t num_groups,
                    const int32_t *group_prefix_blocks, int32_t num_blocks,
                    uint16_t *k_pool, uint16_t *v_pool, uint32_t *free_bits,
                    const uint16_t *k_new, const uint16_t *v_new, int32_t *deficit,
                    const int32_t *req_type, int64_t active_blocks, int64_t threshold_blocks);

int orc_kv_append(int32_t num_reqs, int32_t Hkv, int32_t d,
                  const int32_t *q_indptr, const int32_t *ctx_len,
                  int32_t *block_table, int32_t max_blocks,
                  const int32_t *group_of, int32_t num_groups,
                  const int32_t *group_prefix_blocks, int32_t num_blocks,
                  uint16_t *k_pool, uint16_t *v_pool, uint32_t *free_bits,
                  const uint16_t *k_new, const uint16_t *v_new, int32_t *deficit) {
  return orc_kv_append_t(num_reqs, Hkv, d, q_indptr, ctx_len, block_table, max_blocks, group_of,
                         num_groups, group_prefix_blocks, num_blocks, k_pool, v_pool, free_bits,
                         k_new, v_new, deficit, nullptr, 0, -1);
}

/* kv_append with the burst-reserve threshold ("set a threshold to limit the KV
 * cache size for running online tasks and active offline tasks while leaving sufficient space
 * for future bursty online tasks"; "allocation fails with NeedsEviction if it would
 * push active-class tokens over threshold_tokens, even when free capacity exists ... incoming
 * online allocations may use the reserve, offline may not").  req_type[i] in {0 online decode,
 * 1 offline prefill, 2 offline decode, 3 online prefill}; active_blocks = blocks of the
 * active classes before this step (the manager step's count); threshold_blocks < 0 = no
 * threshold.  Checks, in order: capacity (need > free -> NEEDS_EVICTION, deficit = need -
 * free); then, if any OFFLINE request needs a block: active + need > threshold ->
 * NEEDS_EVICTION with deficit = active + need - threshold (reading R35).  Nothing changes on
 * any error. */
int orc_kv_append_t(int32_t num_reqs, int32_t Hkv, int32_t d,
                    const int32_t *q_indptr, const int32_t *ctx_len,
                    int32_t *block_table, int32_t max_blocks,
                    const int32_t *group_of, int32_t num_groups,
                    const int32_t *group_prefix_blocks, int32_t num_blocks,
                    uint16_t *k_pool, uint16_t *v_pool, uint32_t *free_bits,
                    const uint16_t *k_new, const uint16_t *v_new, int32_t *deficit,
                    const int32_t *req_type, int64_t active_blocks, int64_t threshold_blocks) {
  Batch b = make_batch(num_reqs, Hkv, Hkv, d, q_indptr, ctx_len, block_table, max_blocks,
                       group_of, num_groups, group_prefix_blocks, num_blocks, 0.0);
  if (deficit) *deficit = 0;
  int st = validate(b, false);
  if (st != ST_OK) return st;
  /* resident positions [0, ctx-q_len) must be allocated; new-position
   * entries must be -1 or a valid id */
  int64_t need = 0, need_offline = 0;
  for (int i = 0; i < num_reqs; ++i) {
    const int64_t need_before = need;
    int ctx = ctx_len[i], start = ctx - q_len_of(b, i);
    if ((ctx + BLOCK - 1) / BLOCK > num_blocks) return ST_CAPACITY;
    for (int blk = 0; blk < (start + BLOCK - 1) / BLOCK; ++blk) {
      int id = block_table[(int64_t)i * max_blocks + blk];
      if (id < 0 || id >= num_blocks) return ST_INVALID;
    }
    int last_counted = -1;
    for (int t = start; t < ctx; ++t) {
      int blk = t / BLOCK;
      int id = block_table[(int64_t)i * max_blocks + blk];
      if (id == -1) {
        if (blk != last_counted) { ++need; last_counted = blk; }
      } else if (id < 0 || id >= num_blocks) {
        return ST_INVALID;
      }
    }
    if (req_type && (req_type[i] == 1 || req_type[i] == 2)) need_offline += need - need_before;
  }
  int64_t free_count = 0;
  for (int blk = 0; blk < num_blocks; ++blk) free_count += (free_bits[blk / 32] >> (blk % 32)) & 1u;
  if (need > free_count) {
    if (deficit) *deficit = (int32_t)(need - free_count);
    return ST_NEEDS_EVICTION;
  }
  if (threshold_blocks >= 0 && need_offline > 0 && active_blocks + need > threshold_blocks) {
    if (deficit) *deficit = (int32_t)(active_blocks + need - threshold_blocks);
    return ST_NEEDS_EVICTION;
  }
  int scan = 0; /* smallest free id is found by a forward scan */
  for (int i = 0; i < num_reqs; ++i) {
    int ctx = ctx_len[i], ql = q_len_of(b, i), start = ctx - ql;
    for (int t = start; t < ctx; ++t) {
      int32_t *entry = &block_table[(int64_t)i * max_blocks + t / BLOCK];
      if (*entry == -1) {
        while (!((free_bits[scan / 32] >> (scan % 32)) & 1u)) ++scan;
        free_bits[scan / 32] &= ~(1u << (scan % 32));
        *entry = scan;
      }
      int64_t row = q_indptr[i] + (t - start);
      for (int h = 0; h < Hkv; ++h) {
        int64_t dst = (((int64_t)*entry * Hkv + h) * BLOCK + t % BLOCK) * d;
        int64_t src = (row * Hkv + h) * d;
        std::memcpy(k_pool + dst, k_new + src, sizeof(uint16_t) * d);
        std::memcpy(v_pool + dst, v_new + src, sizeof(uint16_t) * d);
      }
    }
  }
  return ST_OK;
}

/* Block classes (S:103 BlockMeta.task_class, plus the two never-evictable
 * states of reading #17). */
enum { BS_FREE = 0, BS_RUNNING_ONLINE = 1, BS_PINNED = 2, BS_ACTIVE_OFFLINE = 3,
       BS_FINISHED_ONLINE = 4, BS_FINISHED_OFFLINE = 5 };

/* priority_of encoded as an order-preserving key
 * (readings #15-#20):
 *   running online / pinned / free -> +inf  (UINT64_MAX, never selected)
 *   rc > 0                         -> priority rc       (code 2*rc, sat. 0xFFFE)
 *   finished online, rc == 0       -> priority 0.5      (code 1)
 *   otherwise (offline, rc == 0)   -> priority 0        (code 0)
 *   key = code << 48 | lat << 16 | (0xFFFF - min(depth, 0xFFFF)). */
int orc_evict_keys(const uint8_t *state, const uint32_t *rc, const uint32_t *lat,
                   const uint16_t *depth, int64_t n, uint64_t *keys) {
  for (int64_t b = 0; b < n; ++b) {
    uint8_t s = state[b];
    if (s > BS_FINISHED_OFFLINE) return ST_INVALID;
    if (s == BS_FREE || s == BS_RUNNING_ONLINE || s == BS_PINNED) {
      keys[b] = UINT64_MAX;
      continue;
    }
    double priority;
    if (rc[b] > 0) priority = (double)rc[b];
    else if (s == BS_FINISHED_ONLINE) priority = 0.5;
    else priority = 0.0;
    double code_d = std::min(2.0 * priority, (double)0xFFFE);
    uint64_t code = (uint64_t)code_d;
    uint64_t dep = depth ? std::min<uint64_t>(depth[b], 0xFFFF) : 0;
    keys[b] = (code << 48) | ((uint64_t)lat[b] << 16) | (0xFFFFull - dep);
  }
  return ST_OK;
}

/* Eviction order ("first consider the priority ... then the last
 * access time"; P:440 free table = priority queue; tie-break by block id
 * S:200): sort evictable blocks by (key, id) ascending, take the first k. */
/* The KV manager's per-iteration metadata pass (§4.2):
 *  1. class transitions (S:161-168 release_request; reading #17 pins): for chain j in list
 *     order, every block id of chain_ids[chain_indptr[j] .. chain_indptr[j+1]) gets
 *     state = chain_state[j] and lat = now (a later chain overrides an earlier one);
 *  2. reference counts (S:154-160 update_references; "how many offline requests
 *     (including current running request) will reuse it"):
 *     recount != 0: rc[b] = number of offline-pool chains p that list b
 *                   (pool_ids[pool_indptr[p] .. pool_indptr[p+1]));
 *     recount == 0 (incremental): rc[b] += #chains of pool_ids that list b (requests that
 *                   joined the pool) - #chains of del_ids that list b (requests that left it);
 *                   a count that would go negative -> INVALID, nothing changed;
 *  3. *n_active = blocks of the active classes ("tokens held by {RunningOnline,
 *     ActiveOffline}"): running online or pinned, or rc > 0 in any resident class
 *     (S:119 a finished block with rc > 0 is classed ActiveOffline; reading #15);
 *  4. keys = orc_evict_keys(state, rc, lat, depth).
 * Validation first (ids in [0, n), states <= 5, monotone indptr); INVALID = nothing changed. */
int orc_manager_step(uint8_t *state, uint32_t *rc, uint32_t *lat, const uint16_t *depth, int64_t n,
                     uint32_t now, int32_t n_chains, const int32_t *chain_indptr,
                     const int32_t *chain_ids, const uint8_t *chain_state, int32_t n_pool,
                     const int32_t *pool_indptr, const int32_t *pool_ids, int32_t recount,
                     int32_t n_del, const int32_t *del_indptr, const int32_t *del_ids,
                     uint64_t *keys, int64_t *n_active) {
  if (n_chains < 0 || n_pool < 0) return ST_INVALID;
  if (n_chains > 0 && chain_indptr[0] != 0) return ST_INVALID;
  for (int32_t j = 0; j < n_chains; ++j) {
    if (chain_indptr[j + 1] < chain_indptr[j] || chain_state[j] > BS_FINISHED_OFFLINE) return ST_INVALID;
    for (int32_t e = chain_indptr[j]; e < chain_indptr[j + 1]; ++e)
      if (chain_ids[e] < 0 || chain_ids[e] >= n) return ST_INVALID;
  }
  if (n_pool > 0 && pool_indptr[0] != 0) return ST_INVALID;
  for (int32_t p = 0; p < n_pool; ++p) {
    if (pool_indptr[p + 1] < pool_indptr[p]) return ST_INVALID;
    for (int32_t e = pool_indptr[p]; e < pool_indptr[p + 1]; ++e)
      if (pool_ids[e] < 0 || pool_ids[e] >= n) return ST_INVALID;
  }
  if (n_del < 0 || (recount && n_del > 0)) return ST_INVALID;
  if (n_del > 0 && del_indptr[0] != 0) return ST_INVALID;
  for (int32_t p = 0; p < n_del; ++p) {
    if (del_indptr[p + 1] < del_indptr[p]) return ST_INVALID;
    for (int32_t e = del_indptr[p]; e < del_indptr[p + 1]; ++e)
      if (del_ids[e] < 0 || del_ids[e] >= n) return ST_INVALID;
  }
  for (int64_t b = 0; b < n; ++b)
    if (state[b] > BS_FINISHED_OFFLINE) return ST_INVALID;
  std::vector<int64_t> rc_new(n);
  for (int64_t b = 0; b < n; ++b) rc_new[b] = recount ? 0 : (int64_t)rc[b];
  for (int32_t p = 0; p < n_pool; ++p)
    for (int32_t e = pool_indptr[p]; e < pool_indptr[p + 1]; ++e) rc_new[pool_ids[e]] += 1;
  for (int32_t p = 0; p < n_del; ++p)
    for (int32_t e = del_indptr[p]; e < del_indptr[p + 1]; ++e) rc_new[del_ids[e]] -= 1;
  for (int64_t b = 0; b < n; ++b)
    if (rc_new[b] < 0 || rc_new[b] > (int64_t)UINT32_MAX) return ST_INVALID;
  /* 1 */
  for (int32_t j = 0; j < n_chains; ++j)
    for (int32_t e = chain_indptr[j]; e < chain_indptr[j + 1]; ++e) {
      state[chain_ids[e]] = chain_state[j];
      lat[chain_ids[e]] = now;
    }
  /* 2 */
  for (int64_t b = 0; b < n; ++b) rc[b] = (uint32_t)rc_new[b];
  /* 3 */
  int64_t act = 0;
  for (int64_t b = 0; b < n; ++b) {
    if (state[b] == BS_FREE) continue;
    if (state[b] == BS_RUNNING_ONLINE || state[b] == BS_PINNED || rc[b] > 0) ++act;
  }
  if (n_active) *n_active = act;
  /* 4 */
  return orc_evict_keys(state, rc, lat, depth, n, keys);
}

int orc_evict_select(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                     int64_t *n_selected) {
  if (n < 0 || k < 0) return ST_INVALID;
  std::vector<std::pair<uint64_t, int32_t>> cand;
  for (int64_t b = 0; b < n; ++b)
    if (keys[b] != UINT64_MAX) cand.emplace_back(keys[b], (int32_t)b);
  std::sort(cand.begin(), cand.end());
  int64_t m = std::min<int64_t>(k, (int64_t)cand.size());
  for (int64_t s = 0; s < m; ++s) out_ids[s] = cand[s].second;
  *n_selected = m;
  return m < k ? ST_EVICTION_SHORT : ST_OK;
}

/* evict_select with apply (SURVEY §8(c) c1.4 "if apply is set, mark the selected blocks
 * free"; P:440 the evicted blocks return to the free table; "victims ... removed").
 * The selection is orc_evict_select's; then, for each selected id, its free bit (bit b%32 of
 * word b/32) is set.  free_bits has ceil(n/32) words; nothing else changes. */
int orc_evict_select_apply(const uint64_t *keys, int64_t n, int64_t k, int32_t *out_ids,
                           int64_t *n_selected, uint32_t *free_bits) {
  int st = orc_evict_select(keys, n, k, out_ids, n_selected);
  if (st != ST_OK && st != ST_EVICTION_SHORT) return st;
  for (int64_t s = 0; s < *n_selected; ++s)
    free_bits[out_ids[s] / 32] |= 1u << (out_ids[s] % 32);
  return st;
}

/* Release blocks to the free pool ("preempts and release the KV cache of the victim
 * request"; S:143-146 removed blocks become free).  Every id must be in [0, num_blocks),
 * currently allocated (free bit clear) and listed once, else INVALID with nothing changed;
 * then each id's free bit is set. */
int orc_release_blocks(uint32_t *free_bits, int32_t num_blocks, const int32_t *ids, int64_t n) {
  std::vector<char> seen(num_blocks > 0 ? num_blocks : 0, 0);
  for (int64_t s = 0; s < n; ++s) {
    int32_t b = ids[s];
    if (b < 0 || b >= num_blocks) return ST_INVALID;
    if ((free_bits[b / 32] >> (b % 32)) & 1u) return ST_INVALID;  /* already free */
    if (seen[b]) return ST_INVALID;                                  /* listed twice */
    seen[b] = 1;
  }
  for (int64_t s = 0; s < n; ++s) free_bits[ids[s] / 32] |= 1u << (ids[s] % 32);
  return ST_OK;
}

/* Group validation only (for boundary tests). */
int orc_validate(int32_t num_reqs, int32_t Hq, int32_t Hkv, int32_t d,
                 const int32_t *q_indptr, const int32_t *ctx_len,
                 const int32_t *block_table, int32_t max_blocks,
                 const int32_t *group_of, int32_t num_groups,
                 const int32_t *group_prefix_blocks, int32_t num_blocks) {
  Batch b = make_batch(num_reqs, Hq, Hkv, d, q_indptr, ctx_len, block_table, max_blocks,
                       group_of, num_groups, group_prefix_blocks, num_blocks, 0.0);
  return validate(b, true);
}

} // extern "C"
