"""Per-step time of the device Adam epoch (fm_epi_adam_steps, CUDA graph of
the epoch) at a BASELINE config: one IRLS moment pass, then R repeats of an
epoch timed with CUDA events on the launching stream; prints the median
microseconds per Adam step.  A/B two builds with FASTMAP_B200_LIB.

    python tools/adam_probe.py c2 fp32 [reps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2505_04612_b200 import _native as N, epipolar as E, scenes
from paper_2505_04612_b200.config import HotPathConfig

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
prec = sys.argv[2] if len(sys.argv) > 2 else "fp32"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
dev = torch.device("cuda")
sc = scenes.generate(scenes.CONFIGS[cfgname], dev)
store = scenes.device_store(sc, dev)
graph, ids = scenes.device_graph(sc, dev)
params = torch.as_tensor(scenes.initial_params(sc, ids), device=dev)
cfg = HotPathConfig()
eng = E.IrlsEngine(store, graph, params, cfg, precision=prec)
eng._ghat()
eng.point_pass(N.FM_PASS_PRUNE | N.FM_PASS_MOMENTS | N.FM_PASS_IRLS, 1e9, 1, 0)
Z = int(eng.buf.tot.cpu().numpy()[1])
steps = cfg.epipolar_epoch_steps
p0 = params.clone()
st = N.stream_handle()


def epoch():
    N.check(eng.lib.fm_epi_adam_steps(
        ctypes.byref(graph.struct()), ctypes.byref(eng.buf.quad), N.ptr(params), N.ptr(eng.adam_m),
        N.ptr(eng.adam_v), 0, steps, cfg.epipolar_lr, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
        2.0 / Z, N.ptr(eng.flag), 1, N.ptr(eng.gscratch), eng.gscratch.numel(), st))


times = []
for r in range(reps + 3):
    params.copy_(p0)
    eng.adam_m.zero_()
    eng.adam_v.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    epoch()
    b.record()
    torch.cuda.synchronize()
    if r >= 3:
        times.append(a.elapsed_time(b) * 1e3 / steps)
N.raise_flag(eng.flag.item())
times.sort()
print(f"{cfgname} {prec} P={graph.n_pairs} N={graph.n_images} adam step median {times[len(times) // 2]:.2f} us "
      f"min {times[0]:.2f} us  params checksum {float(params.double().sum()):.17g}")
