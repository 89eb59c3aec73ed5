"""Per-SM dispatch rank vs duration of the C2 hot-pass blocks (needs the
-DFM_HOT_TRACE build, see tools/trace_probe.py):
    FASTMAP_B200_LIB=build_variants/trace.so python tools/trace_rank.py"""
import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
spec = scenes.CONFIGS["c2"]
sc = scenes.generate(spec, dev); store = scenes.device_store(sc, dev); graph, ids = scenes.device_graph(sc, dev)
params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision="fp32"); eng._ghat()
mode = N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED
lib = N.lib(); lib.fm_debug_hot_trace.argtypes = [ctypes.c_void_p]
buf = np.zeros((16384, 4), dtype=np.uint64)
for rep in range(3):
    lib.fm_debug_hot_trace(buf.ctypes.data)
    eng.buf.n_active[0].fill_(1)
    eng.point_pass(mode, 0.01, 0, 0)
    torch.cuda.synchronize()
    buf[:] = 0
    lib.fm_debug_hot_trace(buf.ctypes.data)
nb = int((buf[:, 3] > 0).sum())
b = buf[:nb].astype(np.int64)
t0 = b[:, 1].min()
st, ex = (b[:, 1] - t0) / 1e3, (b[:, 3] - t0) / 1e3
dur = ex - st
sm = b[:, 0]
rank = np.zeros(nb, int)
for k in range(148):
    idx = np.flatnonzero(sm == k)
    order = idx[np.argsort(st[idx], kind="stable")]
    rank[order] = np.arange(len(order))
print("blocks", nb, "span", ex.max())
for r in range(rank.max() + 1):
    m = rank == r
    print(f"rank {r}: n {m.sum()} start med {np.median(st[m]):.2f} dur med {np.median(dur[m]):.1f} min {dur[m].min():.1f} max {dur[m].max():.1f} exit med {np.median(ex[m]):.1f}")
# blockIdx groups
for q in range(4):
    m = (np.arange(nb) // 148) == q
    print(f"blockIdx wave-rank {q}: dur med {np.median(dur[m]):.1f}")
# correlation of duration with block's item count? print slowest blocks' idx
sl = np.argsort(-dur)[:10]
print("slowest", [(int(i), int(sm[i]), int(rank[i]), round(float(dur[i]),1)) for i in sl])
span = ex.max()
for t in np.linspace(0, span, 24)[:-1]:
    act = ((st <= t) & (ex > t))
    print(f"   t={t:6.1f} us resident blocks {int(act.sum()):5d}  SMs busy {len(np.unique(sm[act])):3d}")
