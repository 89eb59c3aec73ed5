"""build_tracks + complete_matches at scale: a synthetic match graph of
n_images images x n_kp keypoints; every image sees a window of global
points, pairs (i, i+1..i+w) share the points both see (so tracks are
consistent), each correspondence kept with probability 0.7.
    python tools/tracks_bench.py [ours|reference] [n_images] [n_kp]
('reference' imports /root/reference here, for a one-off CPU timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

which = sys.argv[1] if len(sys.argv) > 1 else "ours"
n_img = int(sys.argv[2]) if len(sys.argv) > 2 else 500
n_kp = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
if which == "reference":
    sys.path.insert(0, "/root/reference/pkg/src")
    from fastmap.model import GeometryClass as GC, ImageInfo, ImagePairMatches as Pair, MatchSet
    from fastmap.tracks import build_tracks, complete_matches
    images = [ImageInfo(i, 0, 640, 480, f"{i}") for i in range(n_img)]
else:
    from tests.test_tracks_gpu import GC, Pair, MS as MatchSet
    from types import SimpleNamespace
    from paper_2505_04612_b200.tracks import build_tracks, complete_matches
    images = [SimpleNamespace(image_id=i) for i in range(n_img)]
rng = np.random.default_rng(0)
# image i sees global points [i*n_kp/4, i*n_kp/4 + n_kp): keypoint k <-> point i*n_kp/4 + perm_i[k]
step = n_kp // 4
perms = [rng.permutation(n_kp) for _ in range(n_img)]
inv = [np.argsort(p) for p in perms]
pairs = []
for i in range(n_img):
    for j in range(i + 1, min(i + 4, n_img)):
        lo = j * step  # points seen by both: [j*step, i*step + n_kp)
        pts = np.arange(lo, i * step + n_kp)
        pts = pts[rng.random(len(pts)) < 0.7]
        ki = inv[i][pts - i * step]
        kj = inv[j][pts - j * step]
        pairs.append(Pair(i, j, GC.FUNDAMENTAL, np.stack([ki, kj], 1).astype(np.int64)))
ms = MatchSet(images=images, keypoints=[np.zeros((n_kp, 2))] * n_img, pairs=pairs)
n_corr = sum(len(p.correspondences) for p in pairs)
if which == "ours":
    complete_matches(build_tracks(ms), ms)  # warm-up (context, module load)
t0 = time.perf_counter()
ts = build_tracks(ms)
t1 = time.perf_counter()
done = complete_matches(ts, ms)
t2 = time.perf_counter()
print({"impl": which, "images": n_img, "pairs": len(pairs), "correspondences": n_corr,
       "tracks": len(ts.tracks), "completed_pairs": len(done.pairs),
       "completed_corr": int(sum(len(p.correspondences) for p in done.pairs)),
       "build_tracks_s": round(t1 - t0, 4), "complete_matches_s": round(t2 - t1, 4)})
