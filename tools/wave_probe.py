"""Per-point cost of the fused pass vs work-item count (wave quantization probe).
    python tools/wave_probe.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig

dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
mode = N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED
cases = [(296, 16, 400), (592, 16, 400), (500, 50, 400), (500, 50, 1600), (2000, 50, 400)]
if len(sys.argv) > 1:
    cases = [tuple(int(x) for x in c.split(",")) for c in sys.argv[1:]]
for n_img, band, ppp in cases:
    spec = scenes.SceneSpec(n_images=n_img, band=band, points_per_pair=ppp)
    sc = scenes.generate(spec, dev)
    store = scenes.device_store(sc, dev)
    graph, ids = scenes.device_graph(sc, dev)
    for prec in ["fp32", "fp64"]:
        params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
        eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec)
        eng._ghat()
        res = {}
        for L in ["auto", "4", "8", "d4", "d8"]:
            os.environ.pop("FM_HOT_DYN", None)
            if L == "auto":
                os.environ.pop("FM_HOT_L", None)
            elif L.startswith("d"):
                os.environ["FM_HOT_DYN"] = "1"
                os.environ["FM_HOT_L"] = L[1:]
            else:
                os.environ["FM_HOT_L"] = L
            eng.buf.n_active[0].fill_(1)
            ts = []
            for k in range(15):
                flush.fill_(k)
                torch.cuda._sleep(200_000)
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(); eng.point_pass(mode, 0.01, 0, 0); b.record()
                torch.cuda.synchronize()
                if k >= 5: ts.append(a.elapsed_time(b))
            t = float(np.median(ts)) * 1e3
            res[f"L{L}_us"] = round(t, 2)
            res[f"L{L}_ps_per_pt"] = round(t * 1e6 / store.n_points, 3)
        os.environ.pop("FM_HOT_L", None)
        os.environ.pop("FM_HOT_DYN", None)

        print(json.dumps({"pairs": store.n_pairs, "ppp": ppp, "items": store.n_items, "prec": prec, **res}), flush=True)
    del eng, store, sc, graph
    torch.cuda.empty_cache()
