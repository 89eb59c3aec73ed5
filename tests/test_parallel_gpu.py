"""The sharded epipolar engine (parallel.ShardedIrlsEngine) on one GPU with
several shards: same schedule, same decisions and the same poses as the
single-store engine and the reference (config 1)."""

import numpy as np
import pytest
import torch

from oracle import fastmap_oracle as O
from tests.helpers import Cfg

pytestmark = pytest.mark.gpu

P_ = pytest.importorskip("paper_2505_04612_b200.parallel")


@pytest.mark.parametrize("world,precision", [(1, "fp64"), (3, "fp64"), (1, "fp32"), (3, "fp32")])
def test_sharded_config1_matches_reference(golden_c1, world, precision):
    """fp64 moments: L1 history within 1e-6; fp32 moments (shifted model, the
    default): within the north-star 1e-4.  Decisions and RRA/RTA identical."""
    g = golden_c1
    dev = torch.device("cuda")
    lengths = g["c1_len"].astype(np.int64)
    ij = g["c1_ij"].astype(np.int64)
    x1 = np.column_stack([g["c1_x1"].astype(np.float64), np.ones(len(g["c1_x1"]))])
    x2 = np.column_stack([g["c1_x2"].astype(np.float64), np.ones(len(g["c1_x2"]))])
    cams = np.zeros_like(ij)
    n = int(ij.max()) + 1
    bounds = P_.partition_pairs(lengths, world)
    shards = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev, precision=precision)
    R = g["c1_R_in"]
    params = torch.as_tensor(np.concatenate([np.concatenate([R[:, :, 0], R[:, :, 1]], 1).ravel(),
                                             g["c1_c_in"].ravel(), [0.0]]), device=dev)
    eng = P_.ShardedIrlsEngine(shards, params, Cfg())
    l1 = eng.run()
    np.testing.assert_allclose(l1, g["c1_l1"], rtol=1e-6 if precision == "fp64" else 1e-4)
    assert [eng.dropped, eng.kept] == list(g["c1_counts"])
    p = params.cpu().numpy()
    rot = O.project_to_so3(O.rot6d_to_matrix(p[:6 * n].reshape(n, 6)))
    cen = p[6 * n:9 * n].reshape(n, 3)
    tol_r, tol_c = (2e-5, 5e-5) if precision == "fp64" else (1e-4, 2e-4)
    assert np.abs(rot - g["c1_R_out"]).max() < tol_r
    assert np.abs(cen - g["c1_c_out"]).max() < tol_c
    ours = O.pose_metrics(rot, cen, g["c1_R_gt"], g["c1_c_gt"])
    ref = O.pose_metrics(g["c1_R_out"], g["c1_c_out"], g["c1_R_gt"], g["c1_c_gt"])
    for k in ("RRA@1", "RRA@3", "RTA@1", "RTA@3"):
        assert ours[k] == ref[k]
    counts = np.concatenate([sh.buf.n_active[0 if True else 1].cpu().numpy()[:sh.graph.n_pairs]
                             for sh in shards])
    active = np.concatenate([sh.store.caller_masks() for sh in shards])
    start = np.concatenate([[0], np.cumsum(lengths)])
    per_pair = np.array([active[start[k]:start[k + 1]].sum() for k in range(len(lengths))])
    assert np.array_equal(per_pair, g["c1_active_count"])
    del counts


def _c1_inputs(g):
    lengths = g["c1_len"].astype(np.int64)
    ij = g["c1_ij"].astype(np.int64)
    x1 = np.column_stack([g["c1_x1"].astype(np.float64), np.ones(len(g["c1_x1"]))])
    x2 = np.column_stack([g["c1_x2"].astype(np.float64), np.ones(len(g["c1_x2"]))])
    R = g["c1_R_in"]
    params = np.concatenate([np.concatenate([R[:, :, 0], R[:, :, 1]], 1).ravel(),
                             g["c1_c_in"].ravel(), [0.0]])
    return lengths, ij, x1, x2, params


def test_nccl_step_chunk_bitwise_single_engine(golden_c1):
    """One shard over a real one-rank NCCL communicator: the graphed chunk
    (local gradient -> ncclAllReduce -> replicated Adam,
    fm_epi_adam_steps_nccl) follows the single-store engine's step (pair_grad +
    image_reduce with Adam) bit for bit."""
    from paper_2505_04612_b200 import epipolar as E
    g = golden_c1
    dev = torch.device("cuda")
    lengths, ij, x1, x2, p0 = _c1_inputs(g)
    n = int(ij.max()) + 1
    cams = np.zeros_like(ij)
    bounds = P_.partition_pairs(lengths, 1)
    comm = P_.NcclComm()
    try:
        sh = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev)
        pa = torch.as_tensor(p0.copy(), device=dev)
        eng = P_.ShardedIrlsEngine(sh, pa, Cfg(), comm=comm)
        assert eng.native_steps
        l1a = eng.run()
        ref = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev)[0]
        pb = torch.as_tensor(p0.copy(), device=dev)
        eng1 = E.IrlsEngine(ref.store, ref.graph, pb, Cfg())
        l1b = eng1.run()
        assert l1a == l1b
        assert torch.equal(pa, pb)
        assert [eng.dropped, eng.kept] == [eng1.dropped, eng1.kept]
    finally:
        comm.close()


def test_nccl_comm_one_rank_collectives():
    comm = P_.NcclComm()
    try:
        t = torch.arange(7, dtype=torch.float64, device="cuda")
        assert torch.equal(comm.allreduce_(t.clone()), t)
        (got,) = comm.allgather(t)
        assert torch.equal(got, t)
    finally:
        comm.close()


def _gloo_worker(rank, world, port, path, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = dict(np.load(path))
        lengths, ij, x1, x2, p0 = _c1_inputs(g)
        n = int(ij.max()) + 1
        bounds = P_.partition_pairs(lengths, world)
        sh = P_.make_shards(x1, x2, lengths, ij, np.zeros_like(ij), n, 1, True, bounds,
                            torch.device("cuda"), ranks=[rank])
        params = torch.as_tensor(p0, device="cuda")
        eng = P_.ShardedIrlsEngine(sh, params, Cfg(), comm=P_.TorchComm())
        l1 = eng.run()
        mask = sh[0].store.caller_masks()
        q.put((rank, l1, params.cpu().numpy(), eng.dropped, eng.kept, mask))
    finally:
        dist.destroy_process_group()


def test_two_ranks_gloo_one_gpu_matches_reference():
    """World 2 (two processes sharing the GPU over gloo, the multi-rank
    schedule's host logic): each rank owns half the image pairs of config 1;
    both end with the same parameters, the reference's decisions, RRA/RTA
    and an ATE within 1e-4."""
    import os
    import socket
    import torch.multiprocessing as mp
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_config1.npz")
    g = dict(np.load(path))
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, l1a, pa, da, ka, ma), (_, l1b, pb, db, kb, mb) = res
    assert np.array_equal(pa, pb) and l1a == l1b and (da, ka) == (db, kb)
    np.testing.assert_allclose(l1a, g["c1_l1"], rtol=1e-4)
    assert [da, ka] == list(g["c1_counts"])
    n = int(g["c1_ij"].max()) + 1
    rot = O.project_to_so3(O.rot6d_to_matrix(pa[:6 * n].reshape(n, 6)))
    cen = pa[6 * n:9 * n].reshape(n, 3)
    ours = O.pose_metrics(rot, cen, g["c1_R_gt"], g["c1_c_gt"])
    ref = O.pose_metrics(g["c1_R_out"], g["c1_c_out"], g["c1_R_gt"], g["c1_c_gt"])
    for k in ("RRA@1", "RRA@3", "RTA@1", "RTA@3"):
        assert ours[k] == ref[k]
    assert abs(ours["ATE"] - ref["ATE"]) < 1e-4
    lengths = g["c1_len"].astype(np.int64)
    active = np.concatenate([ma, mb])
    start = np.concatenate([[0], np.cumsum(lengths)])
    per_pair = np.array([active[start[k]:start[k + 1]].sum() for k in range(len(lengths))])
    assert np.array_equal(per_pair, g["c1_active_count"])



def test_peer_exchange_two_ranks_one_gpu_bitwise_sharded_reference(golden_c1):
    """The fused reduce + exchange + Adam over peer memory
    (fm_epi_adam_steps_peer): two ranks in this process, each driven by its
    own thread on its own stream, exchange their blocks' gradient components
    through each other's buffers inside the kernel.  Both ranks end with the
    same parameters, bit for bit the two-shard engine that sums the shards'
    packed gradients in rank order (parallel.ShardedIrlsEngine, two shards,
    one process), and the reference's decisions / RRA / RTA."""
    import threading
    g = golden_c1
    dev = torch.device("cuda")
    lengths, ij, x1, x2, p0 = _c1_inputs(g)
    n = int(ij.max()) + 1
    cams = np.zeros_like(ij)
    bounds = P_.partition_pairs(lengths, 2)
    ref_shards = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev)
    p_ref = torch.as_tensor(p0.copy(), device=dev)
    ref = P_.ShardedIrlsEngine(ref_shards, p_ref, Cfg())
    l1_ref = ref.run()
    shards = P_.make_shards(x1, x2, lengths, ij, cams, n, 1, True, bounds, dev)
    comms = P_.PeerComm.local_group(shards[0].graph.struct(), 2, dev, max_blocks=64)
    out = [None, None]

    def worker(r):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            p = torch.as_tensor(p0.copy(), device=dev)
            eng = P_.ShardedIrlsEngine([shards[r]], p, Cfg(), comm=comms[r])
            assert eng.native_steps
            l1 = eng.run()
            torch.cuda.synchronize()
            out[r] = (l1, p.cpu().numpy(), eng.dropped, eng.kept)

    errors = []

    def guarded(r):
        try:
            worker(r)
        except BaseException as exc:  # noqa: BLE001 - reported below
            errors.append(exc)
            comms[r].reducer.barrier.abort()

    threads = [threading.Thread(target=guarded, args=(r,)) for r in range(2)]
    try:
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=600)
    finally:
        for c in comms:
            c.close()
    assert not errors, errors
    (la, pa, da, ka), (lb, pb, db, kb) = out
    assert np.array_equal(pa, pb) and la == lb and (da, ka) == (db, kb)
    assert la == l1_ref
    assert np.array_equal(pa, p_ref.cpu().numpy())
    assert [da, ka] == list(g["c1_counts"])
    rot = O.project_to_so3(O.rot6d_to_matrix(pa[:6 * n].reshape(n, 6)))
    cen = pa[6 * n:9 * n].reshape(n, 3)
    ours = O.pose_metrics(rot, cen, g["c1_R_gt"], g["c1_c_gt"])
    refm = O.pose_metrics(g["c1_R_out"], g["c1_c_out"], g["c1_R_gt"], g["c1_c_gt"])
    for key in ("RRA@1", "RRA@3", "RTA@1", "RTA@3"):
        assert ours[key] == refm[key]


def test_peer_sum_two_ranks_one_gpu():
    """fm_peer_sum_f64 with two ranks sharing the GPU (one thread + stream
    each): every exchange returns the rank-order sum on both ranks."""
    import threading
    comms = P_.PeerSum.local_group(3, 2)
    vals = [np.random.default_rng(r).normal(size=(50, 3)) for r in range(2)]
    out = [[], []]

    def worker(r):
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            for k in range(50):
                t = torch.as_tensor(vals[r][k], device="cuda").contiguous()
                comms[r].allreduce_(t)
                out[r].append(t.cpu().numpy())
            comms[r].check()

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    try:
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
    finally:
        for c in comms:
            c.close()
    want = vals[0] + vals[1]
    assert np.array_equal(np.stack(out[0]), want) and np.array_equal(np.stack(out[1]), want)


def _ipc_worker(rank, world, port, path, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g = dict(np.load(path))
        lengths, ij, x1, x2, p0 = _c1_inputs(g)
        n = int(ij.max()) + 1
        bounds = P_.partition_pairs(lengths, world)
        sh = P_.make_shards(x1, x2, lengths, ij, np.zeros_like(ij), n, 1, True, bounds,
                            torch.device("cuda"), ranks=[rank])
        comm = P_.PeerComm.from_process_group(sh[0].graph.struct(), torch.device("cuda"))
        try:
            params = torch.as_tensor(p0, device="cuda")
            eng = P_.ShardedIrlsEngine(sh, params, Cfg(), comm=comm)
            l1 = eng.run()
        finally:
            comm.close()
        q.put((rank, l1, params.cpu().numpy(), eng.dropped, eng.kept))
    finally:
        dist.destroy_process_group()


def test_peer_exchange_two_processes_cuda_ipc(golden_c1):
    """The multi-process form of the fused exchange: two processes (gloo
    only for the 64-byte CUDA IPC handles and the pass scalars), each
    mapping the other's exchange buffers (fm_ipc_open_handle) and running
    fm_epi_adam_steps_peer with system-scope release/acquire.  Both end bitwise
    equal to the two-shard engine in one process."""
    import os
    import socket
    import torch.multiprocessing as mp
    g = golden_c1
    path = os.path.join(os.path.dirname(__file__), "golden", "golden_config1.npz")
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, la, pa, da, ka), (_, lb, pb, db, kb) = res
    assert np.array_equal(pa, pb) and la == lb and (da, ka) == (db, kb)
    lengths, ij, x1, x2, p0 = _c1_inputs(g)
    n = int(ij.max()) + 1
    bounds = P_.partition_pairs(lengths, 2)
    ref_sh = P_.make_shards(x1, x2, lengths, ij, np.zeros_like(ij), n, 1, True, bounds,
                            torch.device("cuda"))
    pr = torch.as_tensor(p0.copy(), device="cuda")
    l1_ref = P_.ShardedIrlsEngine(ref_sh, pr, Cfg()).run()
    assert la == l1_ref and np.array_equal(pa, pr.cpu().numpy())
    assert [da, ka] == list(g["c1_counts"])
