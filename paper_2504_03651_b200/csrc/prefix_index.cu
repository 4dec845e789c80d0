// prefix_index.cu — block-granular prefix index and batch grouping, host
// code of libkvattn.  It produces the batch descriptor's group_of / group_prefix_blocks that the
// cascade path (a3) consumes, from token ids:
//   * "Prefix caching ... reduce the recomputation of prefix tokens" (§2.3) and the
//     offline pool's shared prompts (Table 1);
//   * SPEC lookup_prefix: the longest RESIDENT cached prefix of whole blocks
//     (sub-block matches are misses); hit blocks' LAT = now;
//   * "prefix_index entries for victims removed" with no dangling entries:
//     removing a block removes the entries below it (a chain is reachable only through its
//     prefix).
// One trie node per cached block; a child is keyed by (parent node, the block's 16 token ids),
// compared exactly (the hash only buckets).  Identical token prefixes therefore map to the
// same node and the same physical block, which is what makes a group's prefix blocks shared.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <unordered_map>
#include <vector>

#include "../../include/kvattn.h"
#include "internal.h"

namespace {
constexpr int kB = 16;

struct Key {
  int32_t parent;
  int32_t tok[kB];
  bool operator==(const Key &o) const {
    return parent == o.parent && std::memcmp(tok, o.tok, sizeof(tok)) == 0;
  }
};
struct KeyHash {
  size_t operator()(const Key &k) const {
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (uint64_t)(uint32_t)k.parent;
    for (int i = 0; i < kB; ++i) {
      h ^= (uint64_t)(uint32_t)k.tok[i] + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
      h *= 0xBF58476D1CE4E5B9ull;
    }
    return (size_t)(h ^ (h >> 31));
  }
};
struct Node {
  Key key;
  int32_t block = -1, depth = 0;
  uint32_t lat = 0;
  std::vector<int32_t> kids;
  bool live = false;
};
}  // namespace

struct kva_prefix_index {
  std::vector<Node> nodes;  // node 0 = root (empty prefix)
  std::vector<int32_t> free_nodes;
  std::unordered_map<Key, int32_t, KeyHash> child;
  std::unordered_map<int32_t, int32_t> node_of_block;
  kva_prefix_index() {
    nodes.resize(1);
    nodes[0].live = true;
    nodes[0].key.parent = -1;
  }
  int32_t find(int32_t parent, const int32_t *tok) const {
    Key k;
    k.parent = parent;
    std::memcpy(k.tok, tok, sizeof(k.tok));
    auto it = child.find(k);
    return it == child.end() ? -1 : it->second;
  }
  // walk the whole blocks of tokens[0, n): node of each matched block (stops at the first miss)
  void walk(const int32_t *tokens, int64_t n, std::vector<int32_t> &path) const {
    path.clear();
    int32_t cur = 0;
    for (int64_t b = 0; (b + 1) * kB <= n; ++b) {
      const int32_t nx = find(cur, tokens + b * kB);
      if (nx < 0) break;
      path.push_back(nx);
      cur = nx;
    }
  }
  void remove_subtree(int32_t v) {
    std::vector<int32_t> st{v};
    while (!st.empty()) {
      const int32_t x = st.back();
      st.pop_back();
      Node &nd = nodes[x];
      for (int32_t c : nd.kids) st.push_back(c);
      child.erase(nd.key);
      node_of_block.erase(nd.block);
      nd.kids.clear();
      nd.live = false;
      free_nodes.push_back(x);
    }
  }
};

static kva_status px_fail(kva_status s, const char *m) { return kva::set_error(s, m); }

extern "C" kva_status kva_prefix_index_create(kva_prefix_index **out) {
  if (!out) return px_fail(KVA_ERR_INVALID, "null out");
  *out = new kva_prefix_index();
  return KVA_OK;
}

extern "C" kva_status kva_prefix_index_destroy(kva_prefix_index *ix) {
  delete ix;
  return KVA_OK;
}

extern "C" kva_status kva_prefix_insert(kva_prefix_index *ix, const int32_t *tokens, int64_t n_tokens,
                                        const int32_t *block_ids, uint32_t now) {
  if (!ix || (n_tokens > 0 && (!tokens || !block_ids)) || n_tokens < 0) return px_fail(KVA_ERR_INVALID, "bad argument");
  const int64_t nb = n_tokens / kB;  // whole blocks only
  // validate first (atomic): an already-cached block must carry the same id; a new block id
  // must not be cached elsewhere
  int32_t cur = 0;
  int64_t b = 0;
  for (; b < nb; ++b) {
    const int32_t nx = ix->find(cur, tokens + b * kB);
    if (nx < 0) break;
    if (ix->nodes[nx].block != block_ids[b]) return px_fail(KVA_ERR_INVALID, "cached prefix block has another id");
    cur = nx;
  }
  for (int64_t j = b; j < nb; ++j) {
    if (block_ids[j] < 0) return px_fail(KVA_ERR_INVALID, "negative block id");
    if (ix->node_of_block.count(block_ids[j])) return px_fail(KVA_ERR_INVALID, "block id already indexed");
    for (int64_t k = b; k < j; ++k)
      if (block_ids[k] == block_ids[j]) return px_fail(KVA_ERR_INVALID, "block id repeated in chain");
  }
  cur = 0;
  for (int64_t j = 0; j < nb; ++j) {
    int32_t nx = ix->find(cur, tokens + j * kB);
    if (nx < 0) {
      if (!ix->free_nodes.empty()) {
        nx = ix->free_nodes.back();
        ix->free_nodes.pop_back();
      } else {
        nx = (int32_t)ix->nodes.size();
        ix->nodes.emplace_back();
      }
      Node &nd = ix->nodes[nx];
      nd.key.parent = cur;
      std::memcpy(nd.key.tok, tokens + j * kB, sizeof(nd.key.tok));
      nd.block = block_ids[j];
      nd.depth = (int32_t)j + 1;
      nd.kids.clear();
      nd.live = true;
      ix->child[nd.key] = nx;
      ix->node_of_block[nd.block] = nx;
      ix->nodes[cur].kids.push_back(nx);
    }
    ix->nodes[nx].lat = now;
    cur = nx;
  }
  return KVA_OK;
}

extern "C" kva_status kva_prefix_lookup(kva_prefix_index *ix, const int32_t *tokens, int64_t n_tokens,
                                        int32_t *out_block_ids, int64_t cap, int64_t *n_hit, uint32_t now) {
  if (!ix || !n_hit || n_tokens < 0 || (n_tokens > 0 && !tokens)) return px_fail(KVA_ERR_INVALID, "bad argument");
  std::vector<int32_t> path;
  ix->walk(tokens, n_tokens, path);
  *n_hit = (int64_t)path.size();
  for (size_t i = 0; i < path.size(); ++i) {
    ix->nodes[path[i]].lat = now;  // S:127 "lat of hit blocks updated to now"
    if ((int64_t)i < cap && out_block_ids) out_block_ids[i] = ix->nodes[path[i]].block;
  }
  return KVA_OK;
}

extern "C" kva_status kva_prefix_remove(kva_prefix_index *ix, const int32_t *block_ids, int64_t n) {
  if (!ix || n < 0 || (n > 0 && !block_ids)) return px_fail(KVA_ERR_INVALID, "bad argument");
  for (int64_t i = 0; i < n; ++i) {
    auto it = ix->node_of_block.find(block_ids[i]);
    if (it == ix->node_of_block.end()) continue;  // already gone (e.g. below an earlier victim)
    const int32_t v = it->second;
    const int32_t par = ix->nodes[v].key.parent;
    auto &k = ix->nodes[par].kids;
    for (size_t j = 0; j < k.size(); ++j)
      if (k[j] == v) {
        k[j] = k.back();
        k.pop_back();
        break;
      }
    ix->remove_subtree(v);
  }
  return KVA_OK;
}

extern "C" kva_status kva_prefix_size(const kva_prefix_index *ix, int64_t *n_blocks) {
  if (!ix || !n_blocks) return px_fail(KVA_ERR_INVALID, "bad argument");
  *n_blocks = (int64_t)ix->node_of_block.size();
  return KVA_OK;
}

extern "C" kva_status kva_group_batch(kva_prefix_index *ix, int32_t R, const int32_t *const *tokens,
                                      const int64_t *n_tokens, const int32_t *prefix_limit_blocks,
                                      int32_t min_blocks, int32_t *group_of, int32_t *group_prefix_blocks,
                                      int32_t *num_groups) {
  if (!ix || R < 0 || !group_of || !num_groups || min_blocks < 1 || (R > 0 && (!tokens || !n_tokens)))
    return px_fail(KVA_ERR_INVALID, "bad argument");
  std::vector<std::vector<int32_t>> paths(R);
  std::vector<int64_t> usable(R, 0);
  for (int32_t i = 0; i < R; ++i) {
    if (n_tokens[i] < 0 || (n_tokens[i] > 0 && !tokens[i])) return px_fail(KVA_ERR_INVALID, "bad tokens");
    ix->walk(tokens[i], n_tokens[i], paths[i]);
    usable[i] = (int64_t)paths[i].size();
    if (prefix_limit_blocks) usable[i] = std::min<int64_t>(usable[i], std::max(0, prefix_limit_blocks[i]));
  }
  // class of a candidate = its trie node at depth min_blocks (identical token prefix)
  std::unordered_map<int32_t, std::vector<int32_t>> cls;
  std::vector<int32_t> order;  // classes in order of first member
  for (int32_t i = 0; i < R; ++i) {
    group_of[i] = -1;
    if (usable[i] < min_blocks) continue;
    const int32_t key = paths[i][min_blocks - 1];
    auto &v = cls[key];
    if (v.empty()) order.push_back(key);
    v.push_back(i);
  }
  int32_t G = 0;
  for (int32_t key : order) {
    const auto &mem = cls[key];
    if (mem.size() < 2) continue;
    int64_t depth = min_blocks, lim = INT64_MAX;
    for (int32_t i : mem) lim = std::min(lim, usable[i]);
    while (depth < lim) {  // deepest node shared by every member
      const int32_t nd = paths[mem[0]][depth];
      bool same = true;
      for (int32_t i : mem) same = same && paths[i][depth] == nd;
      if (!same) break;
      ++depth;
    }
    for (int32_t i : mem) group_of[i] = G;
    if (group_prefix_blocks) group_prefix_blocks[G] = (int32_t)depth;
    ++G;
  }
  *num_groups = G;
  return KVA_OK;
}

// Nested grouping (multi-level cascade, NEXT-4): level l groups requests whose first
// level_min_blocks[l] blocks are the same entries (thresholds strictly increasing); a level-l
// group's prefix is the deepest entry all its members share (capped by every usable_i); a
// group whose prefix does not extend its parent's is dropped (its members stay in the parent);
// group_parent links each group to the nearest kept group above it.  Groups are numbered
// level by level, in order of first member, so parents precede children.
extern "C" kva_status kva_group_batch_nested(kva_prefix_index *ix, int32_t R, const int32_t *const *tokens,
                                             const int64_t *n_tokens, const int32_t *prefix_limit_blocks,
                                             int32_t n_levels, const int32_t *level_min_blocks,
                                             int32_t *group_of, int32_t *group_prefix_blocks,
                                             int32_t *group_parent, int32_t *num_groups) {
  if (!ix || R < 0 || !group_of || !num_groups || n_levels < 1 || !level_min_blocks ||
      (R > 0 && (!tokens || !n_tokens)))
    return px_fail(KVA_ERR_INVALID, "bad argument");
  for (int l = 0; l < n_levels; ++l)
    if (level_min_blocks[l] < 1 || (l > 0 && level_min_blocks[l] <= level_min_blocks[l - 1]))
      return px_fail(KVA_ERR_INVALID, "level_min_blocks must be >= 1 and strictly increasing");
  std::vector<std::vector<int32_t>> paths(R);
  std::vector<int64_t> usable(R, 0);
  for (int32_t i = 0; i < R; ++i) {
    if (n_tokens[i] < 0 || (n_tokens[i] > 0 && !tokens[i])) return px_fail(KVA_ERR_INVALID, "bad tokens");
    ix->walk(tokens[i], n_tokens[i], paths[i]);
    usable[i] = (int64_t)paths[i].size();
    if (prefix_limit_blocks) usable[i] = std::min<int64_t>(usable[i], std::max(0, prefix_limit_blocks[i]));
  }
  std::vector<int32_t> cur(R, -1);  // deepest kept group of each request so far
  int32_t G = 0;
  for (int l = 0; l < n_levels; ++l) {
    const int32_t m = level_min_blocks[l];
    std::unordered_map<int32_t, std::vector<int32_t>> cls;
    std::vector<int32_t> order;
    for (int32_t i = 0; i < R; ++i) {
      if (usable[i] < m) continue;
      const int32_t key = paths[i][m - 1];
      auto &v = cls[key];
      if (v.empty()) order.push_back(key);
      v.push_back(i);
    }
    std::vector<std::pair<int32_t, int32_t>> assign;  // (request, group) applied after the level
    for (int32_t key : order) {
      const auto &mem = cls[key];
      if (mem.size() < 2) continue;
      int64_t depth = m, lim = INT64_MAX;
      for (int32_t i : mem) lim = std::min(lim, usable[i]);
      while (depth < lim) {
        const int32_t nd = paths[mem[0]][depth];
        bool same = true;
        for (int32_t i : mem) same = same && paths[i][depth] == nd;
        if (!same) break;
        ++depth;
      }
      const int32_t par = cur[mem[0]];  // every member shares the level above (identical prefix)
      if (par >= 0 && group_prefix_blocks && depth <= group_prefix_blocks[par]) continue;  // no own blocks
      if (group_prefix_blocks) group_prefix_blocks[G] = (int32_t)depth;
      if (group_parent) group_parent[G] = par;
      for (int32_t i : mem) assign.emplace_back(i, G);
      ++G;
    }
    for (auto &a : assign) cur[a.first] = a.second;
  }
  for (int32_t i = 0; i < R; ++i) group_of[i] = cur[i];
  *num_groups = G;
  return KVA_OK;
}
