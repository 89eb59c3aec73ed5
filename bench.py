"""Benchmark of the FastMap B200 hot path (BASELINE.json metric).

A step = one fused point-pair pass (residual + prune + L1 + IRLS-weighted W
moments + linearisation gradient terms: the heaviest pass of irls_refine,
ref/epipolar.py:280-310) over the whole synthetic workload, plus the scalar
all-reduce (Z, L1) that irls_refine needs per pass when N > 1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c4|c5]
  python bench.py --impl reference ...     # CPU oracle port on the host cores

Workload at N=1: BASELINE configs[1] (C2: 500 images, 25,000 image pairs,
10,000,000 point pairs), generated on the device.  N>1 (torchrun, one rank
per GPU, NCCL): every rank holds its own C2-sized shard (weak scaling); the
value is all ranks' point pairs / max-over-ranks device time.

The L2 (126 MB) is flushed between timed steps (256 MB write + 256 MB read, outside the
events); inputs (161 MB) are larger than L2 anyway.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "point-pair residual+grad evals/sec (fraction of HBM roofline); SfM optimize time s"
UNIT = "point pairs/s"
BYTES_PER_POINT = 16.0 + 1.0 / 8.0      # fp32 (x1, y1, x2, y2) + 1 mask bit (read)
BYTES_PER_PAIR = 72.0 + 36 * 8 + 8 + 4 + 8 + 4 + 4 + 4 + 4  # ghat in, fp64 W moments/L1/count out, indices


def ncu_traffic(config, precision):
    """DRAM bytes (read + write) per launch of the timed pass, from the
    committed ncu --set full capture of the same kernel and config
    (profiles/traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return float(json.load(open(p))[config][precision]["dram_bytes"])
    except Exception:
        return None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML
    every 5 ms; nvidia-smi fallback)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._ready = threading.Event()
        self._t = None

    def _run_nvml(self):
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        self._ready.set()
        while not self._stop.is_set():
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.samples.append((float(sm), float(mx), int(rs)))
            self._stop.wait(0.0002)

    def _run_smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        bits = [0x8, 0x40, 0x20, 0x4]
        self._ready.set()
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().split(",")
                rs = sum(b for b, v in zip(bits, out[2:]) if v.strip().lower() == "active")
                self.samples.append((float(out[0]), float(out[1]), rs))
            except Exception:
                pass
            self._stop.wait(0.1)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            self._run_smi()
        finally:
            self._ready.set()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=30)  # NVML initialised: sampling covers the timed region
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for name, bit in self.REASONS.items()
                          if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # FM_DIST_BACKEND=gloo: functional check of the multi-rank path with
        # several ranks sharing one GPU (NCCL refuses duplicate devices)
        backend = os.environ.get("FM_DIST_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
        dist.init_process_group(backend)
    if torch.cuda.is_available():
        local = local % torch.cuda.device_count()
    return world, rank, local


# ------------------------------------------------------------ reference arm
def _ref_worker(args):
    x1, x2, lengths, ghat, th = args
    from oracle import fastmap_oracle as O
    flat = O.FlatPairs(np.column_stack([x1, np.ones(len(x1))]),
                       np.column_stack([x2, np.ones(len(x2))]), lengths)
    out = O.point_pass(flat, ghat, threshold=th)
    return float(out["l1"].sum())


def cpu_sample(spec, n_pairs_sample):
    """A bounded prefix of the workload on the host (fp32 coordinates)."""
    import torch
    from paper_2505_04612_b200 import scenes
    device = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    sc = scenes.generate(spec, device, pair_slice=slice(0, n_pairs_sample))
    ids = np.arange(spec.n_images)
    params = scenes.initial_params(sc, ids, refine_focal=True)
    from oracle import fastmap_oracle as O
    ij = sc["ij"]
    gh = O.pair_forward(params, spec.n_images, ij[:, 0], ij[:, 1], np.zeros(len(ij), int),
                        np.zeros(len(ij), int), True)["ghat"]
    return (sc["x1"].cpu().numpy().astype(np.float64), sc["x2"].cpu().numpy().astype(np.float64),
            sc["lengths"], gh)


def time_cpu_pass(spec, n_pairs_sample, procs, repeats=1):
    """Oracle port of the fused pass on a sample, sharded over `procs`
    processes; returns (point pairs/s, seconds, points)."""
    import multiprocessing as mp
    x1, x2, lengths, gh = cpu_sample(spec, n_pairs_sample)
    P = len(lengths)
    bounds = np.linspace(0, P, procs + 1).astype(int)
    start = np.concatenate([[0], np.cumsum(lengths)])
    jobs = [(x1[start[a]:start[b]], x2[start[a]:start[b]], lengths[a:b], gh[a:b], 0.01)
            for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    ctx = mp.get_context("fork")
    best = None
    with ctx.Pool(len(jobs)) as pool:
        pool.map(_ref_worker, jobs[:1])  # warm the workers
        for _ in range(repeats):
            t0 = time.perf_counter()
            pool.map(_ref_worker, jobs)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
    Z = int(lengths.sum())
    return Z / best, best, Z


def run_reference(args, spec, world, rank):
    if rank != 0:
        return
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    procs = len(os.sched_getaffinity(0))
    n_pairs_sample = min(spec.n_pairs, max(procs * 10, int(1.5e6 // spec.points_per_pair)))
    vals = []
    import multiprocessing as mp
    x1, x2, lengths, gh = cpu_sample(spec, n_pairs_sample)
    P = len(lengths)
    bounds = np.linspace(0, P, procs + 1).astype(int)
    start = np.concatenate([[0], np.cumsum(lengths)])
    jobs = [(x1[start[a]:start[b]], x2[start[a]:start[b]], lengths[a:b], gh[a:b], 0.01)
            for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
    Z = int(lengths.sum())
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            pool.map(_ref_worker, jobs)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                vals.append(dt)
    t = float(np.mean(vals))
    v = Z / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config.upper()} prefix sample", "pass": "L1+prune+IRLS W"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": procs, "kind": "port",
                             "sample": f"{Z} point pairs ({P} image pairs) of {args.config.upper()} "
                                       f"per step, numpy oracle (oracle/fastmap_oracle.py) "
                                       f"point_pass sharded over {procs} processes"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- our arm
def run_ours(args, spec, world, rank, local):
    import ctypes

    import torch
    import torch.distributed as dist

    from paper_2505_04612_b200 import _native as N
    from paper_2505_04612_b200 import epipolar as E
    from paper_2505_04612_b200 import scenes

    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if args.strong:
        # strong scaling: the config's image pairs split into contiguous
        # ranges over the ranks; each rank generates only its own range
        lo, hi = spec.n_pairs * rank // world, spec.n_pairs * (rank + 1) // world
        scene = scenes.generate(spec, device, pair_slice=slice(lo, hi))
    else:
        # weak scaling: one config-sized shard per rank (distinct seeds)
        spec_r = scenes.SceneSpec(**{**spec.__dict__, "seed": spec.seed + rank})
        scene = scenes.generate(spec_r, device)
    store = scenes.device_store(scene, device)
    graph, ids = scenes.device_graph(scene, device)
    params = torch.as_tensor(scenes.initial_params(scene, ids), device=device)
    stream = torch.cuda.Stream(device)
    Z = store.n_points
    P = store.n_pairs
    lib = N.lib()
    with torch.cuda.stream(stream):
        eng = E.IrlsEngine(store, graph, params, args.cfg, precision=args.precision)
        eng._ghat()
    mode = N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=device)  # 256 MB, read back clean
    scal = torch.zeros(2, dtype=torch.float64, device=device)
    sync_bytes = 0

    def one_pass():
        eng.point_pass(mode, 0.01, 0, 0)

    def reduce_scalars():
        scal[0] = eng.buf.l1[:P].sum()
        scal[1] = eng.buf.n_active[0][:P].sum().double()
        if world > 1:
            dist.all_reduce(scal)

    # first pass sets the counts used by SKIP_DROPPED and the steady-state mask
    with torch.cuda.stream(stream):
        eng.buf.n_active[0].fill_(1)
        one_pass()
    torch.cuda.synchronize()

    def timed(k_steps, with_flush=True):
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k_steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k_steps)]
        with torch.cuda.stream(stream):
            for k in range(k_steps):
                if with_flush:
                    # evict the store from L2: write 256 MB, then read another
                    # 256 MB so L2 ends up holding clean lines (no dirty
                    # write-back charged to the timed pass)
                    flush.fill_(k & 0xFF)
                    flush_rd.sum()
                # keep the GPU busy until the host has queued the pass, so the
                # events bracket device work only (not host launch latency)
                torch.cuda._sleep(400_000)
                starts[k].record(stream)
                one_pass()
                ends[k].record(stream)
                reduce_scalars()
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in zip(starts, ends)]

    timed(args.warmup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed(args.steps)
    ms_step = float(np.mean(ms))
    t_max = torch.tensor([ms_step], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_step = float(t_max.item())
    Z_all = torch.tensor([Z], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(Z_all)
    value = float(Z_all.item()) / (ms_step * 1e-3)

    # roofline of the dominant kernel (the pass) from the same events
    bytes_launch = BYTES_PER_POINT * Z + BYTES_PER_PAIR * P
    hbm, hbm_kind = peaks()
    achieved = bytes_launch / (ms_step * 1e-3) / 1e9

    # --------------------------------------------------------------- e2e
    # through the C ABI with HOST buffers: pinned host store columns -> H2D,
    # pass, per-pair results -> D2H, every step.
    h_x1 = store.x1.cpu().pin_memory()
    h_x2 = store.x2.cpu().pin_memory()
    h_act = store.active.cpu().pin_memory()
    outs = eng.buf.outputs()
    h_outs = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
    h2d = sum(t.numel() * t.element_size() for t in (h_x1, h_x2, h_act))
    d2h = sum(t.numel() * t.element_size() for t in h_outs)

    def e2e_steps(k_steps):
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s0.record(stream)
            for _ in range(k_steps):
                store.x1.copy_(h_x1, non_blocking=True)
                store.x2.copy_(h_x2, non_blocking=True)
                store.active.copy_(h_act, non_blocking=True)
                one_pass()
                for h, o in zip(h_outs, outs):
                    h.copy_(o, non_blocking=True)
            s1.record(stream)
        torch.cuda.synchronize()
        return s0.elapsed_time(s1) / k_steps

    e2e_steps(2)
    e2e_ms = e2e_steps(max(3, min(args.steps, 10)))
    t_e2e = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_ms = float(t_e2e.item())

    # ------------------------------------------- SfM optimize time (rank 0)
    extra = {}
    if not args.skip_optimize and world > 1:
        # config 3 with the 16 random starts split over the ranks, and the
        # rank-0 scene's irls_refine with its point pairs sharded over the
        # ranks (NCCL all-reduce of the per-image gradient per Adam step)
        tr = translation_bench(device, stream, sharded=True)
        ep = sharded_irls_bench(spec, args, device, stream, world, rank)
        if rank == 0:
            extra["sfm_optimize"] = {"translation_sharded_over_ranks": world, **tr, **ep}
    if rank == 0 and not args.skip_optimize:
        params0 = torch.as_tensor(scenes.initial_params(scene, ids), device=device)
        store.reset_active()
        with torch.cuda.stream(stream):
            eng2 = E.IrlsEngine(store, graph, params0, args.cfg, precision=args.precision)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            l1h = eng2.run()
            torch.cuda.synchronize()
            t_irls = time.perf_counter() - t0
        extra.setdefault("sfm_optimize", {}).update(
            {"irls_refine_s": t_irls, "l1_history": l1h, "dropped_pairs": eng2.dropped,
             "active_pairs": eng2.kept, "schedule": "3 prune rounds x 3 IRLS x 100 Adam steps"})
        if world == 1:
            extra["sfm_optimize"].update(translation_bench(device, stream))

    # ---------------------------------------------------- CPU baseline
    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        procs = 1
        try:
            from threadpoolctl import threadpool_limits
            threadpool_limits(1)
        except Exception:
            pass
        n_s = max(64, int(1.0e6 // spec.points_per_pair))
        v_cpu, t_cpu, z_cpu = time_cpu_pass(spec, n_s, procs)
        cpu = {"value": v_cpu, "unit": UNIT, "cores": procs, "kind": "port",
               "sample": f"{z_cpu} point pairs ({n_s} image pairs) prefix of {args.config.upper()}, "
                         f"oracle/fastmap_oracle.py point_pass, single process, {t_cpu:.2f} s"}

    launches = args.steps * (1 + (1 if store.n_items > store.n_pairs else 0))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": ("f64 (residual, W moments, prune decisions) on f32 coordinates"
                      if args.precision == "fp64" else
                      "f32 W moments (shifted model) + f64 residual on f32 coordinates"),
            "data": "synthetic (device-generated ring scene, random-perturbed poses)",
            "config": {"workload": f"{args.config.upper()}: {spec.n_images} images, "
                                   + (f"{spec.n_pairs} image pairs / {spec.n_pairs * spec.points_per_pair} "
                                      f"point pairs split over {world} GPU(s)" if args.strong else
                                      f"{P} image pairs, {Z} point pairs per GPU")
                                   + f" (band {spec.band}, {spec.points_per_pair} pts/pair)",
                       "pass": "fused L1 + prune + IRLS W moments (irls_refine rounds 1-2 pass)",
                       "precision": args.precision,
                       "l2": "flushed between steps (256 MB write + 256 MB read, outside the events) and inputs > L2",
                       "parallelism": f"dp{world} (point pairs sharded by image pair)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": ncu_traffic(args.config, args.precision),
                         "peak_kind": hbm_kind,
                         "algorithmic_bytes_per_launch": bytes_launch},
            "cpu_baseline": cpu,
            "e2e": {"value": world * Z / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            **extra,
        }
        print(json.dumps(line), flush=True)


def sharded_irls_bench(spec, args, device, stream, world, rank):
    """irls_refine of the rank-0 C2 scene with its image pairs split into
    contiguous point-balanced ranges over the ranks (parallel.ShardedIrlsEngine:
    local passes, one all-reduce of the packed gradient per Adam step)."""
    import torch
    import torch.distributed as dist
    from paper_2505_04612_b200 import parallel as P_
    from paper_2505_04612_b200 import scenes
    from paper_2505_04612_b200.store import PairGraph, PointPairStore
    with torch.cuda.stream(stream):
        sc = scenes.generate(spec, device)  # every rank: the same (rank-0) scene
        lengths = sc["lengths"]
        b = P_.partition_pairs(lengths, world)
        start = np.concatenate([[0], np.cumsum(lengths)])
        lo, hi = int(b[rank]), int(b[rank + 1])
        ij = sc["ij"]
        ids = np.unique(ij)
        ii, jj = np.searchsorted(ids, ij[:, 0]), np.searchsorted(ids, ij[:, 1])
        store = PointPairStore.from_device(sc["x1"][start[lo]:start[hi]], sc["x2"][start[lo]:start[hi]],
                                           lengths[lo:hi], device=device)
        zeros = np.zeros(hi - lo, dtype=np.int64)
        graph = PairGraph(ii[lo:hi], jj[lo:hi], zeros, zeros, len(ids), 1, True, device=device)
        del sc
        params = torch.as_tensor(scenes.initial_params(scenes.generate_poses(spec), ids), device=device)
        eng = P_.ShardedIrlsEngine([P_.Shard(store, graph, args.precision)], params, args.cfg,
                                   comm=P_.TorchComm())
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        l1h = eng.run()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"irls_refine_sharded_s": float(t.item()), "irls_sharded_l1_history": l1h,
            "irls_sharded_over_ranks": world, "irls_sharded_pairs_rank0": hi - lo}


def translation_bench(device, stream, sharded=False):
    """BASELINE configs[2]: 16 batched inits, 2k nodes / 200k edges, 6000
    steps each + merge + final 6000-step run (ref/translation.py:169-186).
    sharded: the starts split over the torch.distributed ranks (collective)."""
    import torch
    from paper_2505_04612_b200 import parallel as P_
    from paper_2505_04612_b200 import translation as T
    from paper_2505_04612_b200.scenes import translation_graph_c3
    n, m = 2000, 200_000
    ei, ej, d, _ = translation_graph_c3(n, m)
    g = T.DirectionGraph(n=n, edges_i=ei, edges_j=ej, directions=d)

    class C:
        translation_lr, translation_steps, translation_inits = 1e-3, 6000, 16
        adam_beta1, adam_beta2, adam_eps = 0.9, 0.999, 1e-8
    class Cw(C):
        translation_steps = 200

    with torch.cuda.stream(stream):
        # warm-up on the same graph and batch shape: device graph upload and
        # the CUDA-graph captures of the batched and the final descent
        if sharded:
            P_.multi_init_align_sharded(g, Cw, seed=0)
        else:
            T.multi_init_align(g, Cw, seed=0)
        torch.cuda.synchronize()
        if sharded:
            import torch.distributed as dist
            dist.barrier()
        t0 = time.perf_counter()
        if sharded:
            centers, loss = P_.multi_init_align_sharded(g, C, seed=0)
        else:
            centers, loss = T.multi_init_align(g, C, seed=0)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if sharded:
            t = torch.tensor([dt], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
    evals = (16 + 1) * 6000 * m
    return {"multi_init_align_s": dt, "translation_loss": loss,
            "translation_config": "C3: 2000 nodes, 200000 edges, 16 inits x 6000 steps + final (after one 200-step warm-up call)",
            "translation_edge_evals_per_s": evals / dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c4", "c5"])
    ap.add_argument("--strong", action="store_true",
                    help="split the config's image pairs over the ranks (strong scaling; "
                         "default: one config-sized shard per rank)")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-optimize", action="store_true")
    ap.add_argument("--precision", default="fp32", choices=["fp64", "fp32"],
                    help="W-moment accumulation of the pass (irls_refine default: fp32)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    from paper_2505_04612_b200 import scenes
    from paper_2505_04612_b200.config import HotPathConfig
    args.cfg = HotPathConfig()
    spec = scenes.CONFIGS[args.config]
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, spec, world, rank)
    else:
        run_ours(args, spec, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
