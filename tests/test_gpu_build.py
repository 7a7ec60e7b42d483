"""-m gpu: hifuse_build_semantic_graphs bit-exact against the oracle's O1
(Alg. 2), on random blocks (empty, ragged, hub columns, many
relations, invalid edges) and on sampled batches of every configuration."""
import numpy as np
import pytest
import torch

import oracle
from synth import CONFIGS, generate_graph, make_batch, random_block, random_schema
from synth.sampler import LayerBlock

from gpu_util import needs_gpu, gpu_build, csr_host, assert_build_equal

pytestmark = [pytest.mark.gpu, needs_gpu]


def _check(blk, et, rs, rd, ranged=False):
    sh, csr, st = gpu_build(blk, et, rs, rd, ranged=ranged)
    ref = oracle.build(oracle.Shape.of(blk, rs, rd), blk, et)
    assert_build_equal(csr_host(sh, csr), ref)
    assert int(st.item()) == ref["status"]


@pytest.mark.parametrize("seed", range(16))
def test_random_blocks(seed):
    rng = np.random.default_rng(1000 + seed)
    T = int(rng.integers(1, 6))
    R = int(rng.integers(1, 40))
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(0, 300, T)
    n_dst = np.minimum(rng.integers(0, 200, T), n_src)
    if not any(n_src[rs[k]] > 0 and n_dst[rd[k]] > 0 for k in range(R)):
        n_src[:] = 50; n_dst[:] = 20
    N = int(rng.integers(0, 5000))
    blk, et = random_block(rng, n_src, n_dst, rs, rd, N, hub_frac=[0, 0.05, 0.5][seed % 3])
    _check(blk, et, rs, rd)


def test_empty_block():
    rng = np.random.default_rng(1)
    blk, et = random_block(rng, [5, 3], [2, 1], [0, 1], [1, 0], 0)
    _check(blk, et, [0, 1], [1, 0])


def test_long_rows_and_huge_column():
    """Rows longer than 32 and a column beyond the shared-memory bitonic cap
    (8192) exercise both long-segment sort paths."""
    rng = np.random.default_rng(2)
    n = 20000
    src = np.zeros(n, np.int32)
    src[::3] = rng.integers(0, 50, len(src[::3]))
    dst = rng.integers(0, 40, n).astype(np.int32)
    blk = LayerBlock(n_src=np.array([100], np.int32), n_dst=np.array([40], np.int32),
                     src_local=src, dst_local=dst, edge_id=rng.integers(0, 10, n),
                     src_global=[np.arange(100)])
    _check(blk, np.zeros(10, np.int32), [0], [0])


def test_invalid_edges_status_and_drop():
    blk = LayerBlock(n_src=np.array([3], np.int32), n_dst=np.array([2], np.int32),
                     src_local=np.array([0, 5, 1, 0, 2], np.int32),
                     dst_local=np.array([0, 0, 9, 1, 1], np.int32),
                     edge_id=np.array([0, 1, 2, 99, 3], np.int64), src_global=[np.arange(3)])
    _check(blk, np.array([0, 0, 0, 7], np.int32), [0], [0])


@pytest.mark.parametrize("seed", range(4))
def test_null_edges(seed):
    """Edge id -1 (capacity padding of the padded GPU sampler, reading C26)
    interleaved with real edges and as a tail: dropped without a status bit,
    bit-exact against the oracle."""
    rng = np.random.default_rng(2000 + seed)
    T, R = 4, 9
    rs, rd = random_schema(rng, T, R)
    n_src = rng.integers(20, 300, T)
    n_dst = np.minimum(rng.integers(5, 200, T), n_src)
    blk, et = random_block(rng, n_src, n_dst, rs, rd, 3000, hub_frac=0.05)
    eid = blk.edge_id.copy()
    eid[rng.random(len(eid)) < 0.2] = -1
    if seed % 2:
        eid[-500:] = -1                                  # a padded tail
    blk = LayerBlock(n_src=blk.n_src, n_dst=blk.n_dst, src_local=blk.src_local,
                     dst_local=blk.dst_local, edge_id=eid, src_global=blk.src_global)
    _check(blk, et, rs, rd)


@pytest.mark.parametrize("key", ["acm", "dblp", "imdb", "freebase", "mag"])
def test_sampled_batches(key):
    cfg = CONFIGS[key]
    g = generate_graph(cfg)
    mb = make_batch(cfg, g, 0)
    rs = np.array([r.src for r in cfg.rels], np.int32)
    rd = np.array([r.dst for r in cfg.rels], np.int32)
    for blk in mb.layers:
        _check(blk, g.edge_type, rs, rd)
        _check(blk, g.edge_type, rs, rd, ranged=True)    # relation-major ids: offsets path


def test_edge_type_offsets():
    from gpu_util import hf, DEV
    rng = np.random.default_rng(5)
    R = 9
    sizes = rng.integers(0, 50, R)
    sizes[3] = 0                                          # an empty relation
    et = np.repeat(np.arange(R, dtype=np.int32), sizes)
    et_d = torch.from_numpy(et).to(DEV)
    off = torch.empty(R + 1, dtype=torch.int64, device=DEV)
    st = torch.zeros(1, dtype=torch.int32, device=DEV)
    hf().edge_type_offsets(et_d, R, off, st)
    assert hf().read_status(st) == 0
    assert np.array_equal(off.cpu().numpy(), np.searchsorted(et, np.arange(R + 1), "left"))
    et2 = et.copy()
    et2[[0, -1]] = et2[[-1, 0]]                           # not sorted any more
    hf().edge_type_offsets(torch.from_numpy(et2).to(DEV), R, off, st)
    assert hf().read_status(st) & 16


def test_random_blocks_relation_major_offsets():
    """Random blocks whose graph-global edge ids are relation-major."""
    for seed in range(6):
        rng = np.random.default_rng(3000 + seed)
        T, R = int(rng.integers(1, 5)), int(rng.integers(1, 30))
        rs, rd = random_schema(rng, T, R)
        n_src = rng.integers(1, 300, T)
        n_dst = np.maximum(np.minimum(rng.integers(0, 200, T), n_src), 1)
        blk, et = random_block(rng, n_src, n_dst, rs, rd, int(rng.integers(1, 5000)))
        order = np.argsort(et, kind="stable")             # relabel ids relation-major
        inv = np.empty_like(order)
        inv[order] = np.arange(len(order))
        blk2 = blk._replace(edge_id=inv[blk.edge_id]) if hasattr(blk, "_replace") else None
        if blk2 is None:
            import dataclasses
            blk2 = dataclasses.replace(blk, edge_id=inv[blk.edge_id].astype(np.int64))
        _check(blk2, et[order], rs, rd)
        _check(blk2, et[order], rs, rd, ranged=True)


def test_deterministic_across_runs():
    rng = np.random.default_rng(9)
    rs, rd = random_schema(rng, 3, 12)
    blk, et = random_block(rng, [400, 300, 200], [100, 80, 60], rs, rd, 8000, hub_frac=0.1)
    a = csr_host(*gpu_build(blk, et, rs, rd)[:2])
    for _ in range(3):
        b = csr_host(*gpu_build(blk, et, rs, rd)[:2])
        assert_build_equal(b, a)
