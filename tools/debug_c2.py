import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig
dev = torch.device("cuda")
for spec in [scenes.SceneSpec(n_images=60, band=10, points_per_pair=100), scenes.CONFIGS["c2"]]:
    for prec in ["fp64", "fp32"]:
        sc = scenes.generate(spec, dev)
        store = scenes.device_store(sc, dev)
        graph, ids = scenes.device_graph(sc, dev)
        params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
        eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec)
        eng._ghat()
        eng.point_pass(N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS, 0.01, 1, 0)
        torch.cuda.synchronize()
        P = graph.n_pairs
        m = eng.buf.mom64 if prec == "fp64" else eng.buf.mom32
        print(spec.n_images, prec, "ghat nan", torch.isnan(eng.buf.ghat0[:, :P]).sum().item(),
              "mom nan", torch.isnan(m[:, :P]).sum().item(), "mom inf", torch.isinf(m[:, :P]).sum().item(),
              "active", eng.buf.n_active[1][:P].sum().item(), "flag", eng.flag.item(), flush=True)
        try:
            l1 = eng.run()
            print("  run ok", l1, eng.dropped)
        except Exception as e:
            print("  run failed", e, "params nan", torch.isnan(params).sum().item())
