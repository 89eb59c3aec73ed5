"""Per-step time of the Adam epoch on BASELINE config 1 (1,225 image pairs,
50 images): the engine irls_refine builds from the fixture's pairs, one
moment pass, then R repeats of a 100-step epoch timed with CUDA events."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2505_04612_b200 import _native as N, epipolar as E, translation as T
from paper_2505_04612_b200.config import HotPathConfig
from paper_2505_04612_b200.store import PairGraph, PointPairStore
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = HotPathConfig()
g, pairs, _ = bench.c1_problem(E.EpipolarPair, T.DirectionGraph)
poses = bench.Poses(g["c1_R_in"].copy(), g["c1_c_in"].copy())
image_ids = sorted({p.i for p in pairs} | {p.j for p in pairs})
state = E.AdjustmentState.from_poses(poses, image_ids, 1, cfg.refine_focal)
dev = N.require_cuda()
ii, jj, ci, cj = E._pair_indices(state, pairs)
store = PointPairStore.from_pairs(pairs, device=dev, sanitize=True)
o = store.order
graph = PairGraph(ii[o], jj[o], ci[o], cj[o], len(image_ids), 1, cfg.refine_focal, device=dev)
params = torch.as_tensor(state.pack(), device=dev)
eng = E.IrlsEngine(store, graph, params, cfg)
eng._ghat()
eng.point_pass(N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS, 0.01, 1, 0)
steps = cfg.epipolar_epoch_steps
p0 = params.clone()
times = []
for r in range(reps + 2):
    params.copy_(p0); eng.adam_m.zero_(); eng.adam_v.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    N.check(eng.lib.fm_epi_adam_steps_z(
        ctypes.byref(graph.struct()), ctypes.byref(eng.buf.quad), N.ptr(params), N.ptr(eng.adam_m),
        N.ptr(eng.adam_v), 0, steps, cfg.epipolar_lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
        N.ptr(eng.buf.tot), N.ptr(eng.flag), 1, N.ptr(eng.gscratch), eng.gscratch.numel(),
        N.stream_handle()))
    b.record(); torch.cuda.synchronize()
    if r >= 2:
        times.append(a.elapsed_time(b) * 1e3 / steps)
N.raise_flag(eng.flag.item())
times.sort()
print(f"c1 P={graph.n_pairs} N={graph.n_images} adam step median {times[len(times) // 2]:.2f} us "
      f"min {times[0]:.2f} us checksum {float(params.sum()):.17g}")
