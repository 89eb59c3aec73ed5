"""Multi-process (gloo, world_size 2, CPU) checks of the sharded epipolar
schedule's algebra: contiguous image-pair shards balanced by point count, and
the all-reduce composition used by parallel.ShardedIrlsEngine -- per-rank
point-pass scalars and per-rank packed gradients summed over ranks equal the
single-process values.  Per-rank compute is the CPU oracle here (the CUDA
shard path is covered by tests/test_parallel_gpu.py on one GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fastmap_oracle as O
from paper_2505_04612_b200.parallel import partition_pairs
from tests.helpers import SimplePair, pairs_from


def test_partition_pairs_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    for P, world in [(1, 1), (7, 2), (100, 8), (5, 8), (1000, 3)]:
        lengths = rng.integers(0, 500, size=P)
        b = partition_pairs(lengths, world)
        assert b[0] == 0 and b[-1] == P and len(b) == world + 1
        assert np.all(np.diff(b) >= 0)
        per = [lengths[b[k]:b[k + 1]].sum() for k in range(world)]
        assert sum(per) == lengths.sum()
        if P >= world:
            assert max(per) - lengths.sum() / world <= lengths.max() + 1
    assert list(partition_pairs(np.array([10, 10, 10, 10]), 2)) == [0, 2, 4]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, g, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pre = "e1_"
    n, cams, rf = (int(x) for x in g[pre + "meta"])
    pairs = pairs_from(g, pre, SimplePair)
    ij = np.asarray(g[pre + "ij"])
    order = np.lexsort((ij[:, 1], ij[:, 0]))
    pairs = [pairs[k] for k in order]
    ij, cc = ij[order], np.asarray(g[pre + "cams"])[order]
    lengths = np.array([len(p.x1) for p in pairs])
    b = partition_pairs(lengths, world)
    lo, hi = b[rank], b[rank + 1]
    mine = pairs[lo:hi]
    params = g[pre + "params"]
    gh = O.pair_forward(params, n, ij[lo:hi, 0], ij[lo:hi, 1], cc[lo:hi, 0], cc[lo:hi, 1], rf)["ghat"]
    flat = O.FlatPairs.from_pairs(mine)
    out = O.point_pass(flat, gh, threshold=0.01)
    scal = torch.tensor([out["n_active"].sum(), (out["n_active"] > 0).sum(), out["l1"].sum()],
                        dtype=torch.float64)
    dist.all_reduce(scal)
    Z = int(scal[0].item())
    loss, grad = O.quad_loss_grad(params, n, ij[lo:hi, 0], ij[lo:hi, 1], cc[lo:hi, 0],
                                  cc[lo:hi, 1], rf, cams, out["W"], Z)
    t = torch.tensor(np.concatenate([grad, [loss]]), dtype=torch.float64)
    dist.all_reduce(t)
    if rank == 0:
        result_q.put((scal.numpy().tolist(), t.numpy()))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_allreduce_equals_single_process(golden_small):
    g = golden_small
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, g, q)) for r in range(2)]
    for p in procs:
        p.start()
    scal, total = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process reference of the same quantities
    pre = "e1_"
    n, cams, rf = (int(x) for x in g[pre + "meta"])
    pairs = pairs_from(g, pre, SimplePair)
    ij, cc = g[pre + "ij"], g[pre + "cams"]
    gh = O.pair_forward(g[pre + "params"], n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf)["ghat"]
    flat = O.FlatPairs.from_pairs(pairs)
    out = O.point_pass(flat, gh, threshold=0.01)
    Z = int(out["n_active"].sum())
    assert scal[0] == Z and scal[1] == int((out["n_active"] > 0).sum())
    np.testing.assert_allclose(scal[2], out["l1"].sum(), rtol=1e-13)
    loss, grad = O.quad_loss_grad(g[pre + "params"], n, ij[:, 0], ij[:, 1], cc[:, 0], cc[:, 1], rf,
                                  cams, out["W"], Z)
    np.testing.assert_allclose(total[-1], loss, rtol=1e-12)
    np.testing.assert_allclose(total[:-1], grad, rtol=1e-10, atol=1e-13 * np.abs(grad).max())


def _gather_worker(rank, world, port, n_inits, result_q):
    """Per-rank stand-in for the translation starts of
    parallel.multi_init_align_sharded: rank r holds the 'runs' of its block
    of starts (here the reference's seeded random starts themselves)."""
    from paper_2505_04612_b200.parallel import TorchComm, gather_blocks, init_blocks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorchComm()
    assert comm.world == world and comm.rank == rank
    b = init_blocks(n_inits, world)
    local = np.stack([np.random.default_rng(7 + k).standard_normal((11, 3))
                      for k in range(b[rank], b[rank + 1])], axis=1).reshape(11, -1, 3)
    runs = gather_blocks(torch.as_tensor(local), b, comm)
    result_q.put((rank, runs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_translation_starts_gather_in_order(world):
    """The all-gather of per-rank start blocks (uneven: 7 starts) assembles
    every run in start order on every rank."""
    n_inits = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, n_inits, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.stack([np.random.default_rng(7 + k).standard_normal((11, 3)) for k in range(n_inits)],
                    axis=1)
    for _, runs in got:
        assert np.array_equal(runs, full)
