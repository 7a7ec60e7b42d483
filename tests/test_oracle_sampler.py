"""-m "not gpu": pins of the GPU-sampler oracle (oracle/sampler.py; SURVEY.md
§8(f) NEXT(1); SPEC.md sample_batch S:L126-143).  The paper fixes no sampler
(it samples "on CPU"), so the pins are the generator's
published test vectors, SPEC's examples, brute force and the statistics of
uniform sampling without replacement."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle.sampler import mix64, rand_upto, floyd, sample_blocks, M64
from synth import CONFIGS, generate_graph, epoch_seeds

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "splitmix64.json")))


def test_splitmix64_published_vectors():
    s = 1234567
    got = [mix64((s + k * 0x9E3779B97F4A7C15) & M64) for k in range(5)]
    assert got == [int(x) for x in GOLD["seed_1234567_first5"]]
    assert mix64(0) == int(GOLD["seed_0_first"], 16)


def star_graph(deg):
    """1 type, 1 relation; vertex 0 has in-neighbours 1..deg."""
    ptr = np.zeros(deg + 2, np.int64)
    ptr[1:] = deg
    return [(ptr, np.arange(1, deg + 1, dtype=np.int32), np.arange(deg, dtype=np.int64))]


def test_spec_star_example():
    """star, center with 5 in-neighbours, fanout [2] -> exactly 2
    edges, both into the center."""
    lay = sample_blocks(star_graph(5), [0], [0], [6], [0], 0, [2], key=7)[0]
    assert len(lay["edge_id"]) == 2 and (lay["dst_local"] == 0).all()
    assert len(set(lay["edge_id"].tolist())) == 2


def test_determinism_and_key_dependence():
    a = sample_blocks(star_graph(40), [0], [0], [41], [0], 0, [5], key=11)[0]
    b = sample_blocks(star_graph(40), [0], [0], [41], [0], 0, [5], key=11)[0]
    assert np.array_equal(a["edge_id"], b["edge_id"])
    diff = sum(not np.array_equal(a["edge_id"],
                                  sample_blocks(star_graph(40), [0], [0], [41], [0], 0, [5],
                                                key=k)[0]["edge_id"]) for k in range(12, 22))
    assert diff >= 9


def test_floyd_subsets_uniform():
    """deg 5, f 2: all C(5,2) = 10 subsets equally likely (chi-square, 9 dof,
    critical value 33.7 at p = 1e-4) and always distinct positions."""
    counts = {c: 0 for c in itertools.combinations(range(5), 2)}
    n = 20000
    for k in range(n):
        s = floyd(mix64(k), 3, 17, 5, 2)
        assert len(set(s)) == 2 and s == sorted(s)
        counts[tuple(s)] += 1
    exp = n / 10
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 33.7, counts


def test_floyd_inclusion_probability():
    """deg 40, f 25: each position kept with probability 25/40."""
    n = 4000
    inc = np.zeros(40)
    for k in range(n):
        inc[floyd(mix64(k + 99), 0, 5, 40, 25)] += 1
    p = 25 / 40
    sd = np.sqrt(n * p * (1 - p))
    assert np.all(np.abs(inc - n * p) < 5 * sd)


def test_rand_upto_range():
    for j in (0, 1, 2, 7, 1000, (1 << 31) - 2):
        vals = [rand_upto(mix64(5), 1, 2, j) for _ in range(1)] + \
               [rand_upto(mix64(q), 1, 2, j) for q in range(200)]
        assert min(vals) >= 0 and max(vals) <= j


@pytest.fixture(scope="module")
def acm():
    cfg = CONFIGS["acm"]
    g = generate_graph(cfg)
    return cfg, g, g.in_csc()


def _check_blocks(cfg, g, layers, seeds, fanout):
    T = cfg.num_types
    rs, rd = g.rel_src, g.rel_dst
    for l, lay in enumerate(layers):
        # message-flow blocks: destinations are a prefix of sources per type
        for t in range(T):
            assert lay["n_src"][t] >= lay["n_dst"][t]
            new = lay["src_gid"][t][lay["n_dst"][t]:]
            assert np.all(np.diff(new) > 0)                     # new sources ascending
            assert len(set(lay["src_gid"][t].tolist())) == len(lay["src_gid"][t])
        if l + 1 < len(layers):
            nxt = layers[l + 1]
            assert np.array_equal(lay["n_dst"], nxt["n_src"])
            for t in range(T):
                assert np.array_equal(lay["src_gid"][t][:lay["n_dst"][t]], nxt["src_gid"][t])
        # no phantom edges: the edge id's endpoints are the block's vertices
        r = g.edge_type[lay["edge_id"]]
        loc = lay["edge_id"] - g.rel_edge_off[r]
        for k in range(len(r)):
            rr = int(r[k])
            assert lay["src_gid"][rs[rr]][lay["src_local"][k]] == g.src[rr][loc[k]]
            assert lay["src_gid"][rd[rr]][lay["dst_local"][k]] == g.dst[rr][loc[k]]
        # per (destination, relation): min(deg, f) distinct edges
        f = fanout[l]
        pairs = {}
        for k in range(len(r)):
            pairs.setdefault((int(rd[r[k]]), int(lay["dst_local"][k]), int(r[k])), []).append(
                int(lay["edge_id"][k]))
        for (t, i, rr), es in pairs.items():
            v = lay["src_gid"][t][i]
            deg = int(np.sum(g.dst[rr] == v))
            assert len(es) == min(deg, f) and len(set(es)) == len(es)
    assert np.array_equal(layers[-1]["src_gid"][cfg.target_type][:len(seeds)], seeds)


def test_blocks_invariants_acm(acm):
    cfg, g, csc = acm
    seeds = epoch_seeds(cfg, 0)[:16]
    layers = sample_blocks(csc, g.rel_src, g.rel_dst, g.counts, seeds, cfg.target_type, [3, 4],
                           key=123)
    _check_blocks(cfg, g, layers, seeds, [3, 4])


def test_full_fanout_is_full_neighbourhood(acm):
    """fanout >= max degree -> every in-edge of the seeds (brute force
    over the global edge list)."""
    cfg, g, csc = acm
    seeds = epoch_seeds(cfg, 0)[:10]
    lay = sample_blocks(csc, g.rel_src, g.rel_dst, g.counts, seeds, cfg.target_type, [10 ** 6],
                        key=5)[0]
    want = set()
    for r in range(g.num_rels):
        if g.rel_dst[r] != cfg.target_type:
            continue
        for k in np.nonzero(np.isin(g.dst[r], seeds))[0]:
            want.add(int(g.rel_edge_off[r] + k))
    assert set(lay["edge_id"].tolist()) == want and len(lay["edge_id"]) == len(want)
