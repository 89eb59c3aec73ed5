"""Per-block timeline of the hot pass (needs build_variants/trace.so built with -DFM_HOT_TRACE:
    python -c "from paper_2505_04612_b200 import build; build.build(force=True, extra=['-DFM_HOT_TRACE'], out='build_variants/trace.so')").
    FASTMAP_B200_LIB=build_variants/trace.so python tools/trace_probe.py [n_img,band,ppp] [fp32|fp64]
TRACE_MODES: comma list of "mix" (default launcher) or a forced L (4, 8, 16)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig
cfg = sys.argv[1] if len(sys.argv) > 1 else "500,50,400"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
dev = torch.device("cuda")
spec = scenes.SceneSpec(**dict(zip(("n_images", "band", "points_per_pair"), (int(x) for x in cfg.split(",")))))
sc = scenes.generate(spec, dev); store = scenes.device_store(sc, dev); graph, ids = scenes.device_graph(sc, dev)
params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec); eng._ghat()
mode = N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED
lib = N.lib(); lib.fm_debug_hot_trace.argtypes = [ctypes.c_void_p]
for tag in os.environ.get("TRACE_MODES", "mix,4,8,16").split(","):
    if tag == "mix":
        os.environ.pop("FM_HOT_L", None)
    else:
        os.environ["FM_HOT_L"] = tag
    buf = np.zeros((16384, 4), dtype=np.uint64)
    lib.fm_debug_hot_trace(buf.ctypes.data)  # previous contents
    eng.buf.n_active[0].fill_(1)
    st_ev, en_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        st_ev.record(); eng.point_pass(mode, 0.01, 0, 0); en_ev.record()
    torch.cuda.synchronize()
    ev_us = st_ev.elapsed_time(en_ev) * 1e3
    buf[:] = 0
    lib.fm_debug_hot_trace(buf.ctypes.data)
    nb = int((buf[:, 3] > 0).sum())
    b = buf[:nb].astype(np.int64)
    t0 = b[:, 1].min()
    st, lp, ex = (b[:, 1] - t0) / 1e3, (b[:, 2] - t0) / 1e3, (b[:, 3] - t0) / 1e3
    dur = ex - st
    sm = b[:, 0]
    last = np.array([ex[sm == k].max() if (sm == k).any() else 0 for k in range(148)])
    first = np.array([st[sm == k].min() if (sm == k).any() else 0 for k in range(148)])
    span = ex.max()
    # block-time integral / (148 SMs x span): how full the machine was on average
    res = np.bincount(sm, minlength=148).max()
    occ = dur.sum() / (148 * span)
    print(f"== {cfg} {prec} {tag}: event {ev_us:.1f} us, blocks {nb}, span {span:.1f} us, "
          f"mean resident blocks/SM {occ:.2f}; block dur med {np.median(dur):.1f} min {dur.min():.1f} max {dur.max():.1f}")
    print(f"   SM first start max {first.max():.1f} us; SM last exit min {last.min():.1f} p10 {np.percentile(last, 10):.1f} "
          f"p50 {np.median(last):.1f} max {last.max():.1f}; epilogue med {np.median(ex - lp):.2f} us")
    for t in np.linspace(0, span, 13)[:-1]:
        act = ((st <= t) & (ex > t))
        print(f"   t={t:6.1f} us resident blocks {int(act.sum()):5d}  SMs busy {len(np.unique(sm[act])):3d}")
