"""Data-parallel epipolar adjustment: point pairs sharded by contiguous
image-pair ranges across GPUs (one process per GPU, NCCL over NVLink).

Every shard owns whole image pairs, so the fused point pass, the W moments,
the prune masks and the per-pair partials stay local.  The exchanges are
(ref/epipolar.py:279-312 schedule):

* after each prune pass: one all-reduce of {Z, kept pairs, L1 sum} (3 doubles);
* per Adam step: one all-reduce of the packed per-image gradient
  (9N + C doubles) and the loss; Adam then runs replicated on every rank
  (identical inputs -> identical parameters, no broadcast).  Over an
  ``NcclComm`` (one shard per process) a 100-step chunk -- gradient kernels,
  ncclAllReduce, Adam -- is one CUDA graph inside the C library
  (fm_epi_adam_steps_nccl); over ``TorchComm`` (gloo, the CPU tests) the
  step is driven from Python.

``ShardedIrlsEngine`` holds one or more local shards; with one shard per
process and a ``torch.distributed`` communicator it is the multi-GPU engine,
with several shards in one process it is the same algebra on one GPU (used to
test the sharded schedule against the single-store engine).
"""

import ctypes

import numpy as np
import torch

from . import _native as N
from .epipolar import IrlsBuffers, prune_thresholds


def partition_pairs(lengths, world):
    """Contiguous image-pair ranges [b_k, b_{k+1}) balanced by point count.

    b_k is the first pair whose preceding points reach k/world of the total,
    so shard point counts differ by at most one pair's points."""
    lengths = np.asarray(lengths, dtype=np.int64)
    P = len(lengths)
    before = np.concatenate([[0], np.cumsum(lengths)])[:-1] if P else np.zeros(0, np.int64)
    total = int(lengths.sum())
    bounds = [0]
    for k in range(1, world):
        b = int(np.searchsorted(before, total * k / world, side="left")) if P else 0
        bounds.append(max(b, bounds[-1]))
    bounds.append(P)
    return np.array(bounds, dtype=np.int64)


class TorchComm:
    """Sum all-reduce over a torch.distributed process group (NCCL/gloo)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def allreduce_(self, t):
        if self.dist.is_initialized() and self.dist.get_world_size(self.group) > 1:
            self.dist.all_reduce(t, group=self.group)
        return t

    @property
    def world(self):
        return self.dist.get_world_size(self.group) if self.dist.is_initialized() else 1

    @property
    def rank(self):
        return self.dist.get_rank(self.group) if self.dist.is_initialized() else 0

    def allgather(self, t):
        """Equal-shaped tensors of every rank, in rank order."""
        if self.world == 1:
            return [t]
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out


class NcclComm:
    """An NCCL communicator of our own over the ranks of a torch.distributed
    group (fm_nccl_comm_init; the unique id goes out through
    broadcast_object_list on any backend).  Its collectives run inside our
    library on the caller's stream, so the sharded Adam chunk -- local
    gradient, ncclAllReduce, replicated Adam -- is one CUDA graph
    (fm_epi_adam_steps_nccl).  Without an initialised process group it is a
    one-rank communicator."""

    native = True

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if on else 1
        self.rank = dist.get_rank(group) if on else 0
        lib = N.lib()
        if not lib.fm_nccl_available():
            raise RuntimeError("NCCL (libnccl.so.2) is not available")
        uid = (ctypes.c_char * 128)()
        if self.rank == 0:
            N.check(lib.fm_nccl_unique_id(uid))
        if self.world > 1:
            obj = [bytes(uid)]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            uid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        N.check(lib.fm_nccl_comm_init(ctypes.byref(h), self.world, uid, self.rank))
        self.handle = h.value

    def allreduce_(self, t):
        assert t.dtype == torch.float64 and t.is_contiguous()
        N.check(N.lib().fm_nccl_allreduce_sum_f64(N.ptr(t), t.numel(), self.handle,
                                                  N.stream_handle()))
        return t

    def allgather(self, t):
        """Equal-shaped float64 tensors of every rank, in rank order."""
        src = t.contiguous().to(torch.float64)
        out = torch.empty((self.world,) + tuple(src.shape), dtype=torch.float64, device=src.device)
        N.check(N.lib().fm_nccl_allgather_f64(N.ptr(src), N.ptr(out), src.numel(), self.handle,
                                              N.stream_handle()))
        return [o.to(t.dtype) for o in out]

    def close(self):
        if self.handle:
            N.check(N.lib().fm_nccl_comm_destroy(self.handle))
            self.handle = None


def _peer_alloc(part_doubles, n_flags):
    """One rank's exchange buffers (whole cudaMalloc allocations, zeroed)."""
    part, ready = ctypes.c_void_p(), ctypes.c_void_p()
    N.check(N.lib().fm_peer_buffers_alloc(part_doubles, n_flags, ctypes.byref(part), ctypes.byref(ready)))
    return part.value, ready.value


def _peer_share(mine, group=None):
    """Exchange the ranks' buffers through CUDA IPC: returns (parts, readies,
    opened) in rank order (own pointers for this rank, mapped peer memory
    for the others)."""
    import torch.distributed as dist
    lib = N.lib()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    hp, hr = (ctypes.c_char * 64)(), (ctypes.c_char * 64)()
    N.check(lib.fm_ipc_get_handle(mine[0], hp))
    N.check(lib.fm_ipc_get_handle(mine[1], hr))
    allh = [None] * world
    dist.all_gather_object(allh, (bytes(hp), bytes(hr)), group=group)
    parts, readies, opened = [], [], []
    for r, (a, b) in enumerate(allh):
        if r == rank:
            parts.append(mine[0])
            readies.append(mine[1])
            continue
        pa, pb = ctypes.c_void_p(), ctypes.c_void_p()
        N.check(lib.fm_ipc_open_handle((ctypes.c_char * 64).from_buffer_copy(a), ctypes.byref(pa)))
        N.check(lib.fm_ipc_open_handle((ctypes.c_char * 64).from_buffer_copy(b), ctypes.byref(pb)))
        parts.append(pa.value)
        readies.append(pb.value)
        opened += [pa.value, pb.value]
    return parts, readies, opened


class PeerSum:
    """In-place sums of up to 32 doubles over the ranks through peer memory
    (fm_peer_sum_f64: one warp publishes, waits for every peer, sums in rank
    order) -- the pass scalars of the sharded step without a separate
    collective library call."""

    native = True

    def __init__(self, n, rank, world, parts, readies, owned, opened=(), system_scope=False):
        self.n, self.rank, self.world = n, rank, world
        dev = torch.device("cuda", torch.cuda.current_device())
        self.part_ptrs = torch.tensor(parts, dtype=torch.int64, device=dev)
        self.ready_ptrs = torch.tensor(readies, dtype=torch.int64, device=dev)
        self.owned, self.opened = owned, list(opened)
        self.system_scope = system_scope
        self.epoch = 0
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)

    @classmethod
    def local_group(cls, n, world):
        bufs = [_peer_alloc(n, 1) for _ in range(world)]
        return [cls(n, r, world, [b[0] for b in bufs], [b[1] for b in bufs], bufs[r])
                for r in range(world)]

    @classmethod
    def from_process_group(cls, n, group=None):
        import torch.distributed as dist
        mine = _peer_alloc(n, 1)
        parts, readies, opened = _peer_share(mine, group)
        return cls(n, dist.get_rank(group), dist.get_world_size(group), parts, readies, mine,
                   opened, system_scope=True)

    def allreduce_(self, t):
        assert t.dtype == torch.float64 and t.is_contiguous() and t.numel() <= self.n
        grp = N.PeerGroup(n_ranks=self.world, rank=self.rank, part=self.part_ptrs.data_ptr(),
                          ready=self.ready_ptrs.data_ptr(), epoch=self.epoch, max_blocks=0,
                          system_scope=int(self.system_scope))
        N.check(N.lib().fm_peer_sum_f64(N.ptr(t), t.numel(), ctypes.byref(grp), N.ptr(self.err),
                                        N.stream_handle()))
        self.epoch += 1
        return t

    def check(self):
        N.raise_flag(self.err.item())

    def close(self):
        lib = N.lib()
        for ptr in self.opened:
            N.check(lib.fm_ipc_close_handle(ptr))
        self.opened = []
        if self.owned:
            N.check(lib.fm_peer_buffers_free(*self.owned))
            self.owned = None


class PeerComm:
    """The sharded step's all-reduce fused into its reduce kernel over peer
    memory (fm_epi_adam_steps_peer): rank r's blocks publish their packed
    gradient components into r's exchange buffer, wait for the same block of
    every peer and sum the ranks' components in rank order inside the kernel
    (no separate collective).  Buffers are whole cudaMalloc allocations
    (fm_peer_buffers_alloc); across processes their CUDA IPC handles go out
    through torch.distributed (fm_ipc_get_handle / fm_ipc_open_handle; the
    peers' memory is then read over NVLink).  ``local_group`` builds several
    ranks inside one process (tests: ranks sharing one GPU, each driven on
    its own stream).  The pass scalars still go through ``allreduce_``
    (torch.distributed), once per prune pass."""

    native = True
    peer = True

    class _LocalReducer:
        """Host rendezvous of in-process ranks (one thread each): sum in rank
        order, the same result for every rank."""

        def __init__(self, world):
            import threading
            self.slots = [None] * world
            self.barrier = threading.Barrier(world, timeout=300)

        def allreduce_(self, rank, t):
            self.slots[rank] = t.cpu()
            self.barrier.wait()
            total = self.slots[0].clone()
            for x in self.slots[1:]:
                total += x
            self.barrier.wait()
            t.copy_(total)
            return t

    def __init__(self, graph_struct, rank, world, part_ptrs, ready_ptrs, owned, max_blocks=0,
                 opened=(), dist_group=None, reducer=None, system_scope=False):
        self.rank, self.world = rank, world
        self.part_ptrs = part_ptrs      # int64 device tensor [world]
        self.ready_ptrs = ready_ptrs    # int64 device tensor [world]
        self.owned = owned              # (part, ready) pointers this object frees
        self.opened = list(opened)      # IPC-mapped peer pointers to close
        self.epoch = 0
        self.max_blocks = max_blocks
        self.dist_group = dist_group
        self.reducer = reducer
        self.system_scope = system_scope
        self.handle = None

    @staticmethod
    def _alloc(gs):
        lib = N.lib()
        return _peer_alloc(lib.fm_peer_part_len(ctypes.byref(gs)), lib.fm_peer_flag_len(ctypes.byref(gs)))

    @classmethod
    def local_group(cls, graph_struct, world, device, max_blocks=0):
        """`world` ranks in this process (one exchange buffer each)."""
        bufs = [cls._alloc(graph_struct) for _ in range(world)]
        parts = torch.tensor([b[0] for b in bufs], dtype=torch.int64, device=device)
        readies = torch.tensor([b[1] for b in bufs], dtype=torch.int64, device=device)
        red = cls._LocalReducer(world)
        return [cls(graph_struct, r, world, parts, readies, bufs[r], max_blocks, reducer=red)
                for r in range(world)]

    @classmethod
    def from_process_group(cls, graph_struct, device, group=None):
        """One rank per process: exchange the buffers' IPC handles."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        mine = cls._alloc(graph_struct)
        parts, readies, opened = _peer_share(mine, group)
        return cls(graph_struct, rank, world,
                   torch.tensor(parts, dtype=torch.int64, device=device),
                   torch.tensor(readies, dtype=torch.int64, device=device), mine,
                   opened=opened, dist_group=group, system_scope=True)

    def struct(self):
        return N.PeerGroup(n_ranks=self.world, rank=self.rank, part=self.part_ptrs.data_ptr(),
                           ready=self.ready_ptrs.data_ptr(), epoch=self.epoch,
                           max_blocks=self.max_blocks, system_scope=int(self.system_scope))

    def allreduce_(self, t):
        import torch.distributed as dist
        if self.reducer is not None:
            return self.reducer.allreduce_(self.rank, t)
        if self.world > 1 and dist.is_initialized():
            dist.all_reduce(t, group=self.dist_group)
        return t

    def close(self):
        lib = N.lib()
        for ptr in self.opened:
            N.check(lib.fm_ipc_close_handle(ptr))
        self.opened = []
        if self.owned:
            N.check(lib.fm_peer_buffers_free(*self.owned))
            self.owned = None


class NoComm:
    world, rank = 1, 0
    native = True  # one rank: the native step chunk with a NULL communicator
    handle = None

    def allreduce_(self, t):
        return t

    def allgather(self, t):
        return [t]


class Shard:
    """One store + pair graph (global image / camera indexing)."""

    def __init__(self, store, graph, precision=None):
        self.store = store
        self.graph = graph
        self.device = store.device
        self.buf = IrlsBuffers(graph.n_pairs, self.device, precision)
        self.pscratch = store.scratch()
        self.gscratch = graph.scratch()
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.grad = torch.zeros(graph.n_params, dtype=torch.float64, device=self.device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)


class ShardedIrlsEngine:
    """irls_refine schedule over sharded point pairs (see module docstring)."""

    def __init__(self, shards, params, cfg, comm=None):
        self.shards = shards
        self.params = params
        self.cfg = cfg
        self.comm = comm or NoComm()
        self.device = params.device
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.aflag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.lib = N.lib()

    def _ghat(self, sh):
        N.check(self.lib.fm_epi_pair_ghat(ctypes.byref(sh.graph.struct()), N.ptr(self.params),
                                          N.ptr(sh.buf.ghat0), N.ptr(sh.flag), N.ptr(sh.gscratch),
                                          sh.gscratch.numel(), N.stream_handle()))

    def _pass(self, sh, mode, th, cur, prev):
        from .epipolar import _pass
        if mode & N.FM_PASS_MOMENTS:
            mode |= sh.buf.flags
        _pass(sh.store, mode, th, ghat=sh.buf.ghat0,
              prev_active=sh.buf.n_active[prev] if (mode & N.FM_PASS_SKIP_DROPPED) else None,
              out=sh.buf.out(cur), scratch=sh.pscratch)

    def _scalars(self, cur, with_l1):
        """{Z, kept pairs, L1 sum, pairs} over the shards and ranks: each
        shard's pass left its fused totals {L1, Z, kept} in buf.tot."""
        s = torch.zeros(4, dtype=torch.float64, device=self.device)
        for sh in self.shards:
            s[0] += sh.buf.tot[1]
            s[1] += sh.buf.tot[2]
            if with_l1:
                s[2] += sh.buf.tot[0]
            s[3] += sh.graph.n_pairs
        self.comm.allreduce_(s)
        return s.cpu().numpy()

    @property
    def native_steps(self):
        """One shard per process over a native communicator: the Adam chunk
        runs as fm_epi_adam_steps_nccl (collective inside the CUDA graph)."""
        return len(self.shards) == 1 and getattr(self.comm, "native", False)

    def _steps_native(self, t0, n_steps, lr, scale):
        cfg = self.cfg
        sh = self.shards[0]
        if getattr(self.comm, "peer", False):
            grp = self.comm.struct()
            N.check(self.lib.fm_epi_adam_steps_peer(
                ctypes.byref(sh.graph.struct()), ctypes.byref(sh.buf.quad), N.ptr(self.params),
                N.ptr(self.m), N.ptr(self.v), t0, n_steps, lr, cfg.adam_beta1, cfg.adam_beta2,
                cfg.adam_eps, scale, N.ptr(self.aflag), ctypes.byref(grp), 1, N.ptr(sh.gscratch),
                sh.gscratch.numel(), N.stream_handle()))
            self.comm.epoch += n_steps
            return
        if getattr(self, "gbuf", None) is None:
            self.gbuf = torch.zeros(sh.graph.n_params + 1, dtype=torch.float64, device=self.device)
        N.check(self.lib.fm_epi_adam_steps_nccl(
            ctypes.byref(sh.graph.struct()), ctypes.byref(sh.buf.quad), N.ptr(self.params),
            N.ptr(self.m), N.ptr(self.v), t0, n_steps, lr, cfg.adam_beta1, cfg.adam_beta2,
            cfg.adam_eps, scale, N.ptr(self.aflag), self.comm.handle, N.ptr(self.gbuf), 1,
            N.ptr(sh.gscratch), sh.gscratch.numel(), N.stream_handle()))

    def _check_flags(self):
        for sh in self.shards:
            N.raise_flag(sh.flag.item())
        N.raise_flag(self.aflag.item())

    def _step(self, t, lr, scale):
        cfg = self.cfg
        total = None
        for sh in self.shards:
            N.check(self.lib.fm_epi_loss_grad(
                ctypes.byref(sh.graph.struct()), ctypes.byref(sh.buf.quad), N.ptr(self.params),
                scale, N.ptr(sh.loss), N.ptr(sh.grad), N.ptr(sh.flag), N.ptr(sh.gscratch),
                sh.gscratch.numel(), N.stream_handle()))
            if total is None:
                total = torch.cat([sh.grad, sh.loss])
            else:
                total += torch.cat([sh.grad, sh.loss])
        self.comm.allreduce_(total)
        # non-finite loss -> device flag (raised at the end of the IRLS
        # iteration, like the graphed single-store engine); no host sync
        bad = ~torch.isfinite(total[-1:])
        self.aflag.masked_fill_(bad & (self.aflag == 0), N.FM_ERR_NONFINITE_LOSS)
        g = total[:-1].contiguous()
        N.check(self.lib.fm_adam_step(N.ptr(self.params), N.ptr(self.m), N.ptr(self.v), N.ptr(g),
                                      self.params.numel(), t, lr, cfg.adam_beta1, cfg.adam_beta2,
                                      cfg.adam_eps, N.ptr(self.aflag), N.stream_handle()))

    def run(self):
        cfg = self.cfg
        l1_history = []
        lr = cfg.epipolar_lr
        cur = 0
        Z = None
        for rnd, th in enumerate(prune_thresholds(cfg)):
            mode = N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS
            if rnd > 0:
                mode |= N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED
            prev, cur = cur, 1 - cur
            for sh in self.shards:
                self._ghat(sh)
                self._pass(sh, mode, th, cur, prev)
            z, kept, l1, p_total = self._scalars(cur, rnd > 0)
            if rnd > 0:
                l1_history.append(float(l1) / Z)
            self._check_flags()
            Z = int(z)
            self.kept = int(kept)
            self.dropped = int(p_total) - self.kept
            if self.kept == 0:
                raise ValueError("all pairs pruned away")
            self.m.zero_()
            self.v.zero_()
            steps = cfg.epipolar_epoch_steps
            for it in range(cfg.irls_iters_between_prunes):
                if it > 0:
                    for sh in self.shards:
                        self._ghat(sh)
                        self._pass(sh, N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED,
                                   0.0, 1 - cur, cur)
                        sh.buf.n_active[cur], sh.buf.n_active[1 - cur] = \
                            sh.buf.n_active[1 - cur], sh.buf.n_active[cur]
                if self.native_steps:
                    self._steps_native(it * steps, steps, lr, 2.0 / Z)
                else:
                    for k in range(steps):
                        self._step(it * steps + k + 1, lr, 2.0 / Z)
                self._check_flags()
            lr /= cfg.lr_decay
        for sh in self.shards:
            self._ghat(sh)
            self._pass(sh, N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED, 0.0, 1 - cur, cur)
            sh.buf.n_active[cur], sh.buf.n_active[1 - cur] = \
                sh.buf.n_active[1 - cur], sh.buf.n_active[cur]
        _, kept, l1, _ = self._scalars(cur, True)
        self._check_flags()
        l1_history.append(float(l1) / Z)
        return l1_history


def make_shards(x1, x2, lengths, ij, cams, n_images, n_cameras, refine_focal, bounds, device,
                precision=None, ranks=None):
    """Build the shards [bounds[k], bounds[k+1]) of a (sorted) pair list.

    x1, x2: host arrays (Z, 2|3); lengths, ij (P, 2) dense image indices,
    cams (P, 2).  ranks selects which shards to build (default: all)."""
    from .store import PairGraph, PointPairStore
    lengths = np.asarray(lengths, dtype=np.int64)
    start = np.concatenate([[0], np.cumsum(lengths)])
    out = []
    for k in (range(len(bounds) - 1) if ranks is None else ranks):
        a, b = int(bounds[k]), int(bounds[k + 1])
        sl = slice(start[a], start[b])
        store = PointPairStore(x1[sl], x2[sl], lengths[a:b], ij[a:b, 0], ij[a:b, 1],
                               device=device, order=np.arange(b - a), sanitize=True)
        graph = PairGraph(ij[a:b, 0], ij[a:b, 1], cams[a:b, 0], cams[a:b, 1], n_images, n_cameras,
                          refine_focal, device=device)
        out.append(Shard(store, graph, precision))
    return out




def init_blocks(n_inits, world):
    """Contiguous blocks of the random starts per rank: rank r runs starts
    [b[r], b[r+1]) (the last ranks may get one fewer)."""
    return np.array([n_inits * r // world for r in range(world + 1)], dtype=np.int64)


def multi_init_align_sharded(graph, cfg, seed=0, comm=None):
    """multi_init_align (ref/translation.py:169-186) with the B random starts
    split into contiguous blocks over the ranks (independent runs,
    no exchange per step).  Each rank descends its block as one batch; one
    all-gather of the final centres (padded to the largest block) assembles
    the B runs in start order on every rank; the merge and the final descent
    then run replicated, so every rank returns the same result.  A run's
    trajectory does not depend on its batch (fm_tr_align), so the result is
    bitwise the single-GPU multi_init_align whenever every block holds >= 2
    starts."""
    from . import translation as T
    comm = comm or TorchComm()
    B = cfg.translation_inits
    if B == 1 or comm.world == 1:
        return T.multi_init_align(graph, cfg, seed=seed)
    dg = T.device_graph(graph)
    b = init_blocks(B, comm.world)
    lo, hi = int(b[comm.rank]), int(b[comm.rank + 1])
    local = T.init_runs(graph, cfg, seed, range(lo, hi), dg) if hi > lo else \
        torch.zeros((graph.n, 0, 3), dtype=torch.float64, device=dg.device)
    runs = gather_blocks(local, b, comm)
    return T.merge_and_finish(graph, cfg, runs, dg)


def gather_blocks(local, b, comm):
    """All-gather per-rank blocks (n, b[r+1]-b[r], k) along dim 1 in rank
    order; blocks are zero-padded to the widest for the collective."""
    width = int(np.max(np.diff(b)))
    pad = torch.zeros((local.shape[0], width) + tuple(local.shape[2:]), dtype=local.dtype,
                      device=local.device)
    pad[:, :local.shape[1]] = local
    parts = comm.allgather(pad)
    return torch.cat([p[:, :int(b[r + 1] - b[r])] for r, p in enumerate(parts)], dim=1)


__all__ = ["partition_pairs", "ShardedIrlsEngine", "Shard", "TorchComm", "NcclComm", "PeerComm", "PeerSum",
           "NoComm",
           "make_shards",
           "init_blocks", "gather_blocks", "multi_init_align_sharded"]
