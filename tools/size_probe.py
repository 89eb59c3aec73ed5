"""Pass time vs problem size (fixed-overhead probe): 500 images, band 50,
points per pair 100..1600; the fused IRLS pass and the L1-only pass."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)  # clean lines after the dirty fill
full = N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED
l1 = N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED
for arg in (sys.argv[1:] or ["100", "200", "400", "800", "1600"]):
    parts = [int(x) for x in arg.split(",")]
    n_img, band, ppp = (500, 50, parts[0]) if len(parts) == 1 else parts
    spec = scenes.SceneSpec(n_images=n_img, band=band, points_per_pair=ppp)
    sc = scenes.generate(spec, dev); store = scenes.device_store(sc, dev); graph, ids = scenes.device_graph(sc, dev)
    params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
    eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision="fp32"); eng._ghat()
    out = {"pairs": store.n_pairs, "ppp": ppp, "points": store.n_points}
    for name, mode in (("full", full), ("l1", l1)):
        eng.buf.n_active[0].fill_(1)
        ts = []
        for k in range(20):
            flush.fill_(k); flush_rd.sum(); torch.cuda._sleep(1_000_000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); eng.point_pass(mode, 0.01, 0, 0); b.record(); torch.cuda.synchronize()
            if k >= 5: ts.append(a.elapsed_time(b))
        out[name + "_us"] = round(float(np.median(ts)) * 1e3, 2)
    print(json.dumps(out), flush=True)
    del eng, store, sc, graph; torch.cuda.empty_cache()
