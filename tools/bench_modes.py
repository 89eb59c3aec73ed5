"""Time the hot point pass in both precisions at C2 (device-generated data)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig

dev = torch.device("cuda")
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
sc = scenes.generate(scenes.CONFIGS[cfgname], dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush_rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)  # 256 MB
for prec in ["fp64", "fp32"]:
    params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
    eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec)
    eng._ghat()
    res = {}
    for name, mode in [("irls", N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED),
                       ("l1_prune_irls", N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED),
                       ("l1", N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED)]:
        eng.buf.n_active[0].fill_(1)
        ts = []
        for k in range(25):
            flush.fill_(k)
            flush_rd.sum()
            torch.cuda._sleep(400_000)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); eng.point_pass(mode, 0.01, 0, 0); b.record()
            torch.cuda.synchronize()
            if k >= 5: ts.append(a.elapsed_time(b))
        res[name] = float(np.median(ts)) * 1e3
    torch.cuda.synchronize()
    t = []
    store.reset_active()
    params.copy_(torch.as_tensor(scenes.initial_params(sc, ids), device=dev))
    eng2 = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec)
    import time
    for rep in range(2):
        store.reset_active()
        params.copy_(torch.as_tensor(scenes.initial_params(sc, ids), device=dev))
        torch.cuda.synchronize(); t0 = time.perf_counter(); eng2.run(); torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    res["irls_refine_s"] = min(t)
    print(json.dumps({"config": cfgname, "precision": prec, "pass_us": res, "points": store.n_points}), flush=True)
