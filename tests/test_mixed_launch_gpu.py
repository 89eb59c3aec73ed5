"""The two forms of the hot pass's mixed launch -- the exact kernels the C2
headline and the C4/C5 passes run -- against the CPU oracle on a scene large
enough to use them (20,000 image pairs of 128 point pairs: one whole L = 4
wave plus a remainder).  FM_HOT_SHORT selects the short form (3 ring stages,
remainder at L = 8; what C2 picks) or the long form (4 stages, remainder at
L = 16; what C4/C5 pick).  Image pairs are sampled from the first wave and
from the remainder; masks and counts bit-exact, L1 / shifted-model terms
within 1e-5, W within 2e-5 of the pair's scale (fp64 moments: 3e-7;
bench.check_pairs, the in-bench check of the timed pass).  Both moment
precisions."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("short", ["1", "0"])
def test_mixed_launch_forms_match_oracle(short, precision, monkeypatch):
    import torch

    import bench
    from paper_2505_04612_b200 import scenes
    from paper_2505_04612_b200.config import HotPathConfig

    monkeypatch.setenv("FM_HOT_SHORT", short)

    class Args:
        cfg = HotPathConfig()

    Args.precision = precision

    dev = torch.device("cuda")
    spec = scenes.SceneSpec(n_images=400, band=50, points_per_pair=128, seed=5)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        sc, store, graph, ids, eng = bench.make_engine(spec, dev, Args())
        assert store.n_items == 20000
        eng._ghat()
        eng.buf.n_active[0].fill_(1)
        eng.point_pass(bench.HOT_MODE(), bench.TH, 0, 0)  # the first pass prunes
        torch.cuda.synchronize()
        sel = np.unique(np.concatenate([np.linspace(0, 18943, 120), np.linspace(18944, 19999, 80)])
                        .astype(np.int64))
        chk = bench.check_pairs(eng, store, bench.HOT_MODE(), sel)
    assert chk["ok"], chk
