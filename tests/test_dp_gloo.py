"""Multi-process (gloo, world_size 2, CPU) check of the data-parallel host
logic: rank batch assignment and the flat-gradient all-reduce reproduce the
single-process average of the same batches' gradients (SURVEY.md §4 DP
equivalence test), with the oracle as the per-rank compute."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from test_oracle_backward import tiny_batch


def _grads(seed, model):
    import oracle.model as om
    layers, et, rs, rd, X0, gid, params, labels, H = tiny_batch(model, seed)
    agg = "gat" if model == "rgat" else "mean"
    fw = om.forward(layers, et, rs, rd, X0, gid, params, agg, H, labels=labels)
    return om.backward(fw, layers, et, params, labels, agg, H), params


def _layout(model):
    from paper_2408_08490_b200.dp import ParamLayout
    return ParamLayout(3, 5, 6, 8, 2 if model == "rgat" else 1, 3, 2, model)


def _worker(rank, world, port, model, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_08490_b200.dp import rank_batches, allreduce_grads
    lay = _layout(model)
    flat = torch.zeros(lay.size, dtype=torch.float64)
    for b in rank_batches(rank, world, 2):          # this rank's batches
        g, _ = _grads(100 + b, model)
        flat += lay.flatten(g, torch.zeros(1, dtype=torch.float64))
    allreduce_grads(flat, world)
    if rank == 0:
        out.put(flat.numpy() / (world * 2))
    dist.destroy_process_group()


@pytest.mark.parametrize("model", ["rgcn", "rgat"])
def test_dp_allreduce_equals_single_process_average(model):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + np.random.default_rng().integers(0, 2000)
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lay = _layout(model)
    ref = torch.zeros(lay.size, dtype=torch.float64)
    for b in range(4):                               # all batches, one process
        g, _ = _grads(100 + b, model)
        ref += lay.flatten(g, torch.zeros(1, dtype=torch.float64))
    np.testing.assert_allclose(got, ref.numpy() / 4, rtol=1e-12, atol=1e-14)


def test_rank_batches_partition_the_epoch():
    from paper_2408_08490_b200.dp import rank_batches
    world, count = 4, 5
    all_ids = sorted(sum((rank_batches(r, world, count) for r in range(world)), []))
    assert all_ids == list(range(world * count))
