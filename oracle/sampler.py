"""GPU-sampler oracle -- TEST INFRASTRUCTURE ONLY (never imported by the
product path; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
may use oracle/).

Plain Python, step by step, of the sampler contract in include/hifuse.h
(Fig. 2 step (1), line 156; SPEC.md
sample_batch):
  * hop h = 0 .. L-1 builds layer L-1-h; its destinations are the seeds (h = 0)
    or the previous hop's sources;
  * every (destination v of type t, relation r into t) pair keeps min(deg, f)
    of v's in-edges of relation r, chosen uniformly without replacement by
    Floyd's algorithm, in ascending in-list position;
  * edges are emitted by destination (type-major, local id), then relation
    ascending, then position;
  * per type the destinations are the first n_dst sources; the new sources
    follow in ascending vertex id (reading C12);
  * randomness: counter-based splitmix64 -- u = mix(mix(mix(hk ^ r) ^ v) ^ j),
    pick in [0, j] = ((u >> 32) * (j + 1)) >> 32, hk = mix(key ^ (0x1000 + h)).
Parity: unpinned by the paper (it fixes no sampler); pinned by SPEC's
examples and by the invariants in tests/test_oracle_sampler.py.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def mix64(z: int) -> int:
    """splitmix64 finaliser (Steele, Lea, Flood 2014), one step."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def rand_upto(hk: int, r: int, v: int, j: int) -> int:
    u = mix64(mix64(mix64(hk ^ r) ^ v) ^ j)
    return ((u >> 32) * (j + 1)) >> 32


def floyd(hk: int, r: int, v: int, deg: int, f: int) -> list:
    """Floyd's algorithm: a uniform f-subset of range(deg) (all if deg <= f)."""
    if deg <= f:
        return list(range(deg))
    chosen = []
    for j in range(deg - f, deg):
        c = rand_upto(hk, r, v, j)
        chosen.append(j if c in chosen else c)
    return sorted(chosen)


def sample_blocks(in_lists, rel_src, rel_dst, type_counts, seeds, target_type, fanout, key):
    """in_lists[r] = (ptr [|V_t(r)|+1], src [E_r] (ids within type s(r)),
    eid [E_r] (global edge ids)).  fanout: per layer, outer first.  Returns
    layers outer first: dict(n_src, n_dst, src_local, dst_local, edge_id,
    src_gid (list per type of ids within type))."""
    T, R, L = len(type_counts), len(rel_src), len(fanout)
    front = [[] for _ in range(T)]
    front[target_type] = [int(v) for v in seeds]
    layers = [None] * L
    for h in range(L):
        f = int(fanout[L - 1 - h])
        hk = mix64((key ^ (0x1000 + h)) & M64)
        n_dst = [len(front[t]) for t in range(T)]
        src_g, dst_l, eids = [], [], []
        for t in range(T):
            for i, v in enumerate(front[t]):
                for r in range(R):
                    if rel_dst[r] != t:
                        continue
                    ptr, src, eid = in_lists[r]
                    b, e = int(ptr[v]), int(ptr[v + 1])
                    for pos in floyd(hk, r, v, e - b, f):
                        src_g.append((int(rel_src[r]), int(src[b + pos])))
                        dst_l.append(i)
                        eids.append(int(eid[b + pos]))
        src_gid = []
        local = []
        for s in range(T):
            known = {v: i for i, v in enumerate(front[s])}
            new = sorted({u for (ss, u) in src_g if ss == s and u not in known})
            lst = list(front[s]) + new
            src_gid.append(lst)
            local.append({v: i for i, v in enumerate(lst)})
        layers[L - 1 - h] = dict(
            n_src=np.array([len(x) for x in src_gid], np.int32),
            n_dst=np.array(n_dst, np.int32),
            src_local=np.array([local[s][u] for (s, u) in src_g], np.int32),
            dst_local=np.array(dst_l, np.int32),
            edge_id=np.array(eids, np.int64),
            src_gid=[np.array(x, np.int64) for x in src_gid])
        front = src_gid
    return layers
