"""Run a few point passes of one mode (for ncu): one_pass.py <mode> <precision> [config]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_04612_b200 import scenes, epipolar as E, _native as N
from paper_2505_04612_b200.config import HotPathConfig
modes = {"irls": N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED,
         "l1": N.FM_PASS_L1 | N.FM_PASS_SKIP_DROPPED,
         "full": N.FM_PASS_L1 | N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS | N.FM_PASS_SKIP_DROPPED}
mode, prec = sys.argv[1], sys.argv[2]
cfg = sys.argv[3] if len(sys.argv) > 3 else "c2"
dev = torch.device("cuda")
spec = scenes.CONFIGS[cfg] if cfg in scenes.CONFIGS else scenes.SceneSpec(
    **dict(zip(("n_images", "band", "points_per_pair"), (int(x) for x in cfg.split(",")))))
sc = scenes.generate(spec, dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
eng = E.IrlsEngine(store, graph, params, HotPathConfig(), precision=prec)
eng._ghat()
eng.buf.n_active[0].fill_(1)
for _ in range(int(os.environ.get("FM_PASSES", "4"))):
    eng.point_pass(modes[mode], 0.01, 0, 0)
torch.cuda.synchronize()
print("done")
