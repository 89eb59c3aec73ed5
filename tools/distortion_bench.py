"""Time search_alpha on the golden scene A (3 levels x 10 candidates x 28 pairs, M = 200)
against the reference's recorded CPU time.   python tools/distortion_bench.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_distortion_gpu import _match_set, _cfg
from paper_2505_04612_b200 import distortion as D
g = np.load("tests/golden/golden_distortion.npz")
ms = _match_set(g, "a_")
pairs = [ms.pairs[k] for k in g["a_ready"]]
D.search_alpha(ms, pairs, _cfg())
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); a = D.search_alpha(ms, pairs, _cfg()); ts.append(time.perf_counter() - t0)
st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
cands = g["a_cands"][0]
jobs = D._jobs(list(cands), ms, pairs, None, None)
t0 = time.perf_counter(); D._jobs(list(cands), ms, pairs, None, None); host = time.perf_counter() - t0
st.record(); D.score_alpha_batch(cands, ms, pairs); en.record(); torch.cuda.synchronize()
print({"alpha": a, "search_alpha_s": min(ts), "ref_search_alpha_s": float(g["a_ref_seconds"]),
       "level_launch_plus_host_ms": st.elapsed_time(en), "host_prep_ms": host * 1e3, "jobs": len(jobs[1])})
from paper_2505_04612_b200 import focal
for pre in ("a_", "b_"):
    ms2 = _match_set(g, pre)
    al = {0: float(g["a_alpha"])} if pre == "a_" else {c: float(a) for c, a in enumerate(g["b_alphas"])}
    focal.undistorted_fundamentals(ms2, al)
    t0 = time.perf_counter(); focal.undistorted_fundamentals(ms2, al); dt = time.perf_counter() - t0
    print({"scene": pre, "undistorted_fundamentals_s": dt, "ref_s": float(g[pre + "fund_seconds"])})
from types import SimpleNamespace
for pre in ("a_", "b_", "c_"):
    ms3 = _match_set(g, pre)
    cams = {}
    for c, (f, a) in enumerate(g[pre + "cam"]):
        im = next(i for i in ms3.images if i.camera_id == c)
        cams[c] = SimpleNamespace(focal=float(f), alpha=float(a), cx=im.width / 2.0, cy=im.height / 2.0,
                                  half_diagonal=0.5 * float(np.hypot(im.width, im.height)))
    focal.apply_calibration(ms3, cams)
    t0 = time.perf_counter(); focal.apply_calibration(ms3, cams); dt = time.perf_counter() - t0
    print({"scene": pre, "apply_calibration_s": dt, "ref_s": float(g[pre + "calib_seconds"])})
