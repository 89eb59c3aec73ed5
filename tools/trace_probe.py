"""Per-block timeline of the hot pass (needs build_variants/trace.so built with -DFM_HOT_TRACE).
    FASTMAP_B200_LIB=build_variants/trace.so python tools/trace_probe.py [n_img,band,ppp] [fp32|fp64]"""
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
for tag in os.environ.get("TRACE_MODES", "plan,4,8").split(","):
    os.environ["FM_HOT_PLAN"] = "1" if tag == "plan" else "0"
    os.environ["FM_HOT_L"] = "4" if tag == "plan" else tag
    eng.buf.n_active[0].fill_(1)
    for _ in range(3):
        eng.point_pass(mode, 0.01, 0, 0)
    torch.cuda.synchronize()
    buf = np.zeros((16384, 4), dtype=np.uint64)
    lib.fm_debug_hot_trace(buf.ctypes.data)
    nb = int(store.n_pairs and len(np.nonzero(buf[:, 2])[0]))
    nb = min(nb, int(np.ceil((store.n_items if tag != "plan" else 1e9) / (32 / int(os.environ["FM_HOT_L"])) / 4)))
    b = buf[:nb].astype(np.int64)
    t0 = b[:, 1].min()
    st, en = (b[:, 1] - t0) / 1e3, (b[:, 2] - t0) / 1e3
    dur = en - st
    print(f"== {cfg} {prec} L/plan={tag}: blocks {nb}, span {en.max():.1f} us, block dur med {np.median(dur):.1f} "
          f"min {dur.min():.1f} max {dur.max():.1f}; first-wave start max {np.sort(st)[min(nb-1, 591)]:.1f}")
    # concurrency histogram: active blocks over time
    ex = (b[:, 3] - t0) / 1e3
    print(f"   epilogue (exit - loop end) med {np.median(ex - en):.2f} max {(ex - en).max():.2f} us; span to exit {ex.max():.1f}")
    for t in np.linspace(0, ex.max(), 12):
        print(f"   t={t:6.1f} us active blocks {int(((st <= t) & (ex > t)).sum())}")
    sm = b[:, 0]
    busy = np.array([ (ex[sm == k].max() - st[sm == k].min()) if (sm == k).any() else 0 for k in range(148)])
    cnt = np.bincount(sm, minlength=148)
    print(f"   per-SM blocks min {cnt.min()} max {cnt.max()}; per-SM span min {busy.min():.1f} max {busy.max():.1f}")
