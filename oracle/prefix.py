"""TEST INFRASTRUCTURE ONLY — brute-force oracle of the prefix index and the batch grouping
(S:125-133 lookup_prefix, S:146 / S:109 removal without dangling entries,
reading #8 for the group precondition).  Plain Python over explicit chains: no trie, no hashing,
no code shared with paper_2504_03651_b200/csrc/prefix_index.cu.

A cached chain is a list of (block token tuple, block id); the cache is the SET of resident
(prefix-of-tokens, block id) facts: block j of a chain is hit-able iff the chain's blocks
0..j are all resident.
"""
from __future__ import annotations

B = 16


class BruteIndex:
    def __init__(self):
        self.entries = {}   # tuple(tokens of blocks 0..j) -> block id of block j

    def insert(self, tokens, block_ids):
        nb = len(tokens) // B
        for j in range(nb):
            key = tuple(tokens[: (j + 1) * B])
            self.entries.setdefault(key, int(block_ids[j]))

    def lookup(self, tokens):
        """longest cached prefix of whole blocks: brute force over every prefix length"""
        hit = []
        for j in range(len(tokens) // B):
            key = tuple(tokens[: (j + 1) * B])
            if key not in self.entries:
                break
            hit.append(self.entries[key])
        return hit

    def remove(self, block_ids):
        gone = set(int(b) for b in block_ids)
        victims = [k for k, v in self.entries.items() if v in gone]
        for vk in victims:  # the victim and every entry whose prefix passes through it
            for k in list(self.entries):
                if len(k) >= len(vk) and k[: len(vk)] == vk:
                    del self.entries[k]

    def size(self):
        return len(self.entries)


def group_batch(index: BruteIndex, token_lists, prefix_limit_blocks=None, min_blocks=1):
    """Definition (include/kvattn.h kva_group_batch): usable_i = min(hit blocks, limit_i);
    candidates (usable >= m) with identical first m blocks form a group when >= 2; the group
    prefix = the longest common whole-block prefix of all members, capped by every usable_i."""
    R = len(token_lists)
    usable = []
    for i, t in enumerate(token_lists):
        u = len(index.lookup(list(t)))
        if prefix_limit_blocks is not None:
            u = min(u, max(0, int(prefix_limit_blocks[i])))
        usable.append(u)
    group_of = [-1] * R
    prefixes = []
    done = set()
    for i in range(R):
        if i in done or usable[i] < min_blocks:
            continue
        head = tuple(token_lists[i][: min_blocks * B])
        mem = [j for j in range(R) if usable[j] >= min_blocks and tuple(token_lists[j][: min_blocks * B]) == head]
        done.update(mem)
        if len(mem) < 2:
            continue
        depth = min(usable[j] for j in mem)
        while depth > min_blocks:
            ref = tuple(token_lists[mem[0]][: depth * B])
            if all(tuple(token_lists[j][: depth * B]) == ref for j in mem):
                break
            depth -= 1
        for j in mem:
            group_of[j] = len(prefixes)
        prefixes.append(depth)
    return group_of, prefixes


def group_batch_nested(index: BruteIndex, token_lists, level_min_blocks, prefix_limit_blocks=None):
    """Definition (include/kvattn.h kva_group_batch_nested) by brute force over token tuples."""
    R = len(token_lists)
    usable = []
    for i, t in enumerate(token_lists):
        u = len(index.lookup(list(t)))
        if prefix_limit_blocks is not None:
            u = min(u, max(0, int(prefix_limit_blocks[i])))
        usable.append(u)
    cur = [-1] * R
    prefixes, parents = [], []
    for m in level_min_blocks:
        assign = []
        done = set()
        for i in range(R):
            if i in done or usable[i] < m:
                continue
            head = tuple(token_lists[i][: m * B])
            mem = [j for j in range(R) if usable[j] >= m and tuple(token_lists[j][: m * B]) == head]
            done.update(mem)
            if len(mem) < 2:
                continue
            depth = min(usable[j] for j in mem)
            while depth > m:
                ref = tuple(token_lists[mem[0]][: depth * B])
                if all(tuple(token_lists[j][: depth * B]) == ref for j in mem):
                    break
                depth -= 1
            par = cur[mem[0]]
            if par >= 0 and depth <= prefixes[par]:
                continue
            g = len(prefixes)
            prefixes.append(depth)
            parents.append(par)
            assign += [(j, g) for j in mem]
        for j, g in assign:
            cur[j] = g
    return cur, prefixes, parents
