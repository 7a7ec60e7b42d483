"""Input generator checks: determinism and the block invariants of the
sampler contract (reading C12)."""
import numpy as np
import pytest

from synth import CONFIGS, generate_graph, make_batch


@pytest.mark.parametrize("key", ["acm", "dblp", "imdb", "freebase"])
def test_batches_are_deterministic_and_well_formed(key):
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    b1 = make_batch(cfg, g, 1)
    b2 = make_batch(cfg, generate_graph(cfg), 1)
    assert len(b1.layers) == cfg.num_layers
    for l1, l2 in zip(b1.layers, b2.layers):
        assert np.array_equal(l1.edge_id, l2.edge_id) and np.array_equal(l1.src_local, l2.src_local)
        r = g.edge_type[l1.edge_id]
        loc = l1.edge_id - g.rel_edge_off[r]
        for e in range(l1.num_edges):
            rr = r[e]
            assert l1.src_global[g.rel_src[rr]][l1.src_local[e]] == g.src[rr][loc[e]]
            assert l1.src_global[g.rel_dst[rr]][l1.dst_local[e]] == g.dst[rr][loc[e]]
            assert l1.dst_local[e] < l1.n_dst[g.rel_dst[rr]]
        # fanout cap per (vertex, relation)
        key2 = r.astype(np.int64) * 10**7 + l1.dst_local
        _, cnt = np.unique(key2 + g.rel_dst[r].astype(np.int64) * 10**9, return_counts=True)
        assert cnt.max() <= max(cfg.fanout)
    for a, b in zip(b1.layers[:-1], b1.layers[1:]):
        assert np.array_equal(a.n_dst, b.n_src)
        for t in range(cfg.num_types):
            assert np.array_equal(a.src_global[t][:a.n_dst[t]], b.src_global[t])
    last = b1.layers[-1]
    assert np.array_equal(last.src_global[cfg.target_type][:last.n_dst[cfg.target_type]], b1.seeds)
