"""The reference's run_pipeline on NOISY_SPEC (acceptance criterion 5), wall
time, unmodified or with install() (our hot path and the section 8(f) stages
on the GPU).  python tools/pipeline_probe.py [ref|dropin]"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import fastmap
from fastmap import metrics, synth
from fastmap.config import PipelineConfig
from fastmap.pipeline import run_pipeline
mode = sys.argv[1] if len(sys.argv) > 1 else "dropin"
if mode == "dropin":
    import paper_2505_04612_b200 as b200
    b200.install(fastmap)
spec = synth.SynthSpec(n_images=30, n_points=500, fov_deg=60.0, alpha=-0.15, noise_px=0.5,
                       outlier_frac=0.02, seed=0)
match_set, gt = synth.generate(spec)
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
    t0 = time.perf_counter()
    scene, report = run_pipeline(match_set, PipelineConfig(), seed=0)
    dt = time.perf_counter() - t0
    table = metrics.evaluate(scene.poses, gt.poses)
    stages = {k: round(v, 3) for k, v in getattr(report, "timings", {}).items()} if hasattr(report, "timings") else str(report)[:600]
    print(json.dumps({"mode": mode, "seconds": dt, "ATE": table["ATE"], "RRA@1": table["RRA@1"],
                      "RTA@3": table["RTA@3"], "stages": stages}))
