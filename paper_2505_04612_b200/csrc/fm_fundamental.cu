// Distortion candidate scoring (SURVEY 8f "next" #4): the robust
// fundamental-matrix fit + epipolar error sum that score_alpha
// (ref/distortion.py:90-126) runs for every (candidate alpha, image pair).
//
// One CTA (128 threads) per job = one (candidate, pair) with M undistorted,
// scaled points.  The job follows estimate_fundamental (ref/twoview.py:58-76):
//   M >= 16: LMedS (ref/twoview.py:79-104) -- Hartley normalisation, 64
//     seeded minimal samples (index table from the host: the reference's own
//     numpy generator calls), per sample the 9x9 normal matrix, its smallest
//     eigenvector (cyclic Jacobi, one thread per sample), rank-2 projection
//     (one-sided Jacobi SVD of the 3x3), residuals of all points, the median
//     per sample (warp radix select), argmin, the 2.5-sigma consensus set,
//     then the least-squares fit on it;
//   M < 16: the least-squares fit on all points (ref/twoview.py:107-123);
// then _refit_on_inliers (ref/twoview.py:48-55), the error sum
// (ref/distortion.py:119-122) and, optionally, the fitted F itself (the
// batched estimate_fundamental of ref/focal.py:72).  A fit whose Frobenius norm is < 1e-15
// reports n_err = 0 (the reference raises and score_alpha skips the pair).
//
// Reductions are block-level in a fixed order (deterministic); medians are
// exact order statistics, so the result differs from numpy only by the
// summation order of centroids / normal matrices (~1e-16 relative).
#include <cmath>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kSamples = 64;  // ref/twoview.py:44 _LMEDS_ITERS

// ---------------------------------------------------------------- 3x3 / 9x9 linear algebra
// Smallest eigenvector of a symmetric 9x9 matrix (cyclic Jacobi; a is destroyed).
__device__ void smallest_eigvec9(double (&a)[9][9], double (&out)[9]) {
  double v[9][9];
  for (int i = 0; i < 9; ++i)
    for (int j = 0; j < 9; ++j) v[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int p = 0; p < 9; ++p) {
      diag += a[p][p] * a[p][p];
      for (int q = p + 1; q < 9; ++q) off += a[p][q] * a[p][q];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < 8; ++p)
      for (int q = p + 1; q < 9; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 9; ++k) {  // columns p, q
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = c * akp - s * akq;
          a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 9; ++k) {  // rows p, q
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = c * apk - s * aqk;
          a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 9; ++k) {
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = c * vkp - s * vkq;
          v[k][q] = s * vkp + c * vkq;
        }
      }
  }
  int best = 0;
  for (int i = 1; i < 9; ++i)
    if (a[i][i] < a[best][best]) best = i;
  for (int k = 0; k < 9; ++k) out[k] = v[k][best];
}

// F <- F with its smallest singular value zeroed (U diag(s0, s1, 0) V^T,
// ref/twoview.py:95-98, :117-119): one-sided Jacobi on the columns, F = W V^T.
__device__ void rank2(double (&F)[9]) {
  double W[3][3], V[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) W[i][j] = F[i * 3 + j], V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = 0; k < 3; ++k) {
          al += W[k][p] * W[k][p];
          be += W[k][q] * W[k][q];
          ga += W[k][p] * W[k][q];
        }
        if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int k = 0; k < 3; ++k) {
          const double wp = W[k][p], wq = W[k][q];
          W[k][p] = c * wp - s * wq;
          W[k][q] = s * wp + c * wq;
          const double vp = V[k][p], vq = V[k][q];
          V[k][p] = c * vp - s * vq;
          V[k][q] = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  int mn = 0;
  double nmin = 1e308;
  for (int j = 0; j < 3; ++j) {
    const double n = W[0][j] * W[0][j] + W[1][j] * W[1][j] + W[2][j] * W[2][j];
    if (n < nmin) nmin = n, mn = j;
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k)
        if (k != mn) acc += W[i][k] * V[j][k];
      F[i * 3 + j] = acc;
    }
}

// ---------------------------------------------------------------- block helpers
template <int N>
__device__ void block_sum(double (&v)[N], double* red /* [kWarps][N] */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x = v[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    v[i] = x;
  }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < N; ++i) red[w * N + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double x = 0.0;
    for (int k = 0; k < kWarps; ++k) x += red[k * N + i];
    v[i] = x;
  }
  __syncthreads();
}

// k-th smallest (0-based) of n non-negative doubles, by one warp: radix
// select on the IEEE bit patterns (monotone for x >= 0), 8 bits per pass.
__device__ double warp_kth(const double* buf, int n, int kth, unsigned* hist /* [256] */) {
  const int lane = threadIdx.x & 31;
  unsigned long long prefix = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = lane; i < 256; i += 32) hist[i] = 0;
    __syncwarp();
    for (int m = lane; m < n; m += 32) {
      const unsigned long long key = (unsigned long long)__double_as_longlong(buf[m]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    // lane l owns bins 8l .. 8l+7
    unsigned own = 0;
    for (int i = 0; i < 8; ++i) own += hist[8 * lane + i];
    unsigned incl = own;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned excl = incl - own;
    const unsigned ball = __ballot_sync(0xffffffffu, (unsigned)kth < incl);
    const int src = __ffs(ball) - 1;
    int digit = 0;
    unsigned below = 0;
    if (lane == src) {
      unsigned cum = excl;
      for (int i = 0; i < 8; ++i) {
        const unsigned h = hist[8 * lane + i];
        if ((unsigned)kth < cum + h) {
          digit = 8 * lane + i;
          below = cum;
          break;
        }
        cum += h;
      }
    }
    digit = __shfl_sync(0xffffffffu, digit, src);
    below = __shfl_sync(0xffffffffu, below, src);
    kth -= (int)below;
    prefix |= (unsigned long long)digit << shift;
    mask |= 255ull << shift;
    __syncwarp();
  }
  return __longlong_as_double((long long)prefix);
}

// np.median of n >= 1 non-negative values (mean of the two middle ones for even n)
__device__ double warp_median(const double* buf, int n, unsigned* hist) {
  if (n & 1) return warp_kth(buf, n, (n - 1) / 2, hist);
  const double a = warp_kth(buf, n, n / 2 - 1, hist);
  const double b = warp_kth(buf, n, n / 2, hist);
  return (a + b) / 2.0;
}

struct Hartley {
  double s1, cx1, cy1, s2, cx2, cy2;
};

struct Shared {
  double F[9];
  double Fk[kSamples][9];
  double med[kSamples];
  double red[kWarps * 45];
  Hartley T;
  unsigned hist[kWarps][256];
  int best, status, count;
  double thr;
};

// Hartley normalisation of the masked points of both views (ref/twoview.py:23-35).
__device__ void hartley(const double2* p1, const double2* p2, const unsigned char* keep, int M,
                        Shared& sh) {
  double v[5] = {0, 0, 0, 0, 0};
  for (int m = threadIdx.x; m < M; m += kThreads) {
    if (keep && !keep[m]) continue;
    const double2 a = p1[m], b = p2[m];
    v[0] += a.x, v[1] += a.y, v[2] += b.x, v[3] += b.y, v[4] += 1.0;
  }
  block_sum<5>(v, sh.red);
  const double n = v[4];
  const double cx1 = v[0] / n, cy1 = v[1] / n, cx2 = v[2] / n, cy2 = v[3] / n;
  double d[2] = {0, 0};
  for (int m = threadIdx.x; m < M; m += kThreads) {
    if (keep && !keep[m]) continue;
    const double2 a = p1[m], b = p2[m];
    d[0] += sqrt((a.x - cx1) * (a.x - cx1) + (a.y - cy1) * (a.y - cy1));
    d[1] += sqrt((b.x - cx2) * (b.x - cx2) + (b.y - cy2) * (b.y - cy2));
  }
  block_sum<2>(d, sh.red);
  if (threadIdx.x == 0) {
    sh.T.s1 = sqrt(2.0) / fmax(d[0] / n, 1e-12);
    sh.T.s2 = sqrt(2.0) / fmax(d[1] / n, 1e-12);
    sh.T.cx1 = cx1, sh.T.cy1 = cy1, sh.T.cx2 = cx2, sh.T.cy2 = cy2;
  }
  __syncthreads();
}

// A row = flatten(x2 x1^T) of the Hartley-normalised homogeneous points
__device__ __forceinline__ void design_row(const Hartley& T, double2 a, double2 b, double (&r)[9]) {
  const double x1[3] = {T.s1 * (a.x - T.cx1), T.s1 * (a.y - T.cy1), 1.0};
  const double x2[3] = {T.s2 * (b.x - T.cx2), T.s2 * (b.y - T.cy2), 1.0};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) r[3 * i + j] = x2[i] * x1[j];
}

// Least-squares fit on the masked points (ref/twoview.py:107-123) -> sh.F,
// sh.status = 0 when the fit is degenerate.
__device__ void fit_fundamental(const double2* p1, const double2* p2, const unsigned char* keep,
                                int M, Shared& sh) {
  hartley(p1, p2, keep, M, sh);
  const Hartley T = sh.T;
  double n45[45];
#pragma unroll
  for (int i = 0; i < 45; ++i) n45[i] = 0.0;
  for (int m = threadIdx.x; m < M; m += kThreads) {
    if (keep && !keep[m]) continue;
    double r[9];
    design_row(T, p1[m], p2[m], r);
    int q = 0;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = i; j < 9; ++j) n45[q++] += r[i] * r[j];
  }
  block_sum<45>(n45, sh.red);
  if (threadIdx.x == 0) {
    double a[9][9];
    int q = 0;
    for (int i = 0; i < 9; ++i)
      for (int j = i; j < 9; ++j) a[i][j] = a[j][i] = n45[q++];
    double f[9];
    smallest_eigvec9(a, f);
    rank2(f);
    // F = T2^T F T1, T = [[s, 0, -s cx], [0, s, -s cy], [0, 0, 1]]
    const double t1[9] = {T.s1, 0.0, -T.s1 * T.cx1, 0.0, T.s1, -T.s1 * T.cy1, 0.0, 0.0, 1.0};
    const double t2[9] = {T.s2, 0.0, -T.s2 * T.cx2, 0.0, T.s2, -T.s2 * T.cy2, 0.0, 0.0, 1.0};
    double g[9], h[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += f[i * 3 + k] * t1[k * 3 + j];
        g[i * 3 + j] = acc;  // F T1
      }
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += t2[k * 3 + i] * g[k * 3 + j];
        h[i * 3 + j] = acc;  // T2^T (F T1)
      }
    double nrm = 0.0;
    for (int i = 0; i < 9; ++i) nrm += h[i] * h[i];
    nrm = sqrt(nrm);
    if (!(nrm >= 1e-15)) {
      sh.status = 0;
    } else {
      for (int i = 0; i < 9; ++i) sh.F[i] = h[i] / nrm;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double epi_abs(const double (&F)[9], double2 a, double2 b) {
  const double y0 = F[0] * a.x + F[1] * a.y + F[2];
  const double y1 = F[3] * a.x + F[4] * a.y + F[5];
  const double y2 = F[6] * a.x + F[7] * a.y + F[8];
  return fabs(b.x * y0 + b.y * y1 + y2);
}

__global__ void __launch_bounds__(kThreads)
fund_score_kernel(const int64_t* __restrict__ job_off, const double2* __restrict__ p1all,
                  const double2* __restrict__ p2all, const int32_t* __restrict__ sample_idx,
                  const int64_t* __restrict__ sample_off, double* __restrict__ err_sum,
                  int32_t* __restrict__ n_err, double* __restrict__ F_out, double* __restrict__ rbuf_all,
                  unsigned char* __restrict__ keep_all) {
  __shared__ Shared sh;
  const int64_t job = blockIdx.x;
  const int64_t off = job_off[job];
  const int M = (int)(job_off[job + 1] - off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (M < 8) {
    if (threadIdx.x == 0) {
      err_sum[job] = 0.0, n_err[job] = 0;
      if (F_out)
        for (int i = 0; i < 9; ++i) F_out[9 * job + i] = NAN;
    }
    return;
  }
  const double2* p1 = p1all + off;
  const double2* p2 = p2all + off;
  double* rbuf = rbuf_all + kWarps * off;  // kWarps x M
  unsigned char* keep = keep_all + off;
  if (threadIdx.x == 0) sh.status = 1;
  __syncthreads();

  if (sample_off[job] >= 0) {
    // ---------------- LMedS (ref/twoview.py:79-104)
    hartley(p1, p2, nullptr, M, sh);
    const Hartley T = sh.T;
    if (threadIdx.x < kSamples) {
      const int32_t* idx = sample_idx + sample_off[job] + 8 * threadIdx.x;
      double a[9][9];
      for (int i = 0; i < 9; ++i)
        for (int j = 0; j < 9; ++j) a[i][j] = 0.0;
      for (int r = 0; r < 8; ++r) {
        const int m = idx[r];
        double row[9];
        design_row(T, p1[m], p2[m], row);
        for (int i = 0; i < 9; ++i)
          for (int j = i; j < 9; ++j) a[i][j] += row[i] * row[j];
      }
      for (int i = 0; i < 9; ++i)
        for (int j = 0; j < i; ++j) a[i][j] = a[j][i];
      double f[9];
      smallest_eigvec9(a, f);
      rank2(f);
      for (int i = 0; i < 9; ++i) sh.Fk[threadIdx.x][i] = f[i];
    }
    __syncthreads();
    // per-sample median residual over all points (in normalised coordinates)
    double* mybuf = rbuf + (int64_t)w * M;
    for (int k = w; k < kSamples; k += kWarps) {
      double F[9];
      for (int i = 0; i < 9; ++i) F[i] = sh.Fk[k][i];
      for (int m = lane; m < M; m += 32) {
        const double2 a = p1[m], b = p2[m];
        const double2 x1 = make_double2(T.s1 * (a.x - T.cx1), T.s1 * (a.y - T.cy1));
        const double2 x2 = make_double2(T.s2 * (b.x - T.cx2), T.s2 * (b.y - T.cy2));
        mybuf[m] = epi_abs(F, x1, x2);
      }
      __syncwarp();
      const double med = warp_median(mybuf, M, sh.hist[w]);
      if (lane == 0) sh.med[k] = med;
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int b = 0;
      for (int k = 1; k < kSamples; ++k)
        if (sh.med[k] < sh.med[b]) b = k;  // first minimum, as np.argmin
      sh.best = b;
    }
    __syncthreads();
    double F[9];
    for (int i = 0; i < 9; ++i) F[i] = sh.Fk[sh.best][i];
    for (int m = threadIdx.x; m < M; m += kThreads) {
      const double2 a = p1[m], b = p2[m];
      const double2 x1 = make_double2(T.s1 * (a.x - T.cx1), T.s1 * (a.y - T.cy1));
      const double2 x2 = make_double2(T.s2 * (b.x - T.cx2), T.s2 * (b.y - T.cy2));
      rbuf[m] = epi_abs(F, x1, x2);
    }
    __syncthreads();
    if (w == 0) {
      // median(rb^2): rb >= 0, so its middle order statistics are those of rb
      double m2;
      if (M & 1) {
        const double x = warp_kth(rbuf, M, (M - 1) / 2, sh.hist[0]);
        m2 = x * x;
      } else {
        const double x = warp_kth(rbuf, M, M / 2 - 1, sh.hist[0]);
        const double y = warp_kth(rbuf, M, M / 2, sh.hist[0]);
        m2 = (x * x + y * y) / 2.0;
      }
      if (lane == 0) {
        const double sigma = 1.4826 * (1.0 + 5.0 / (M - 8)) * sqrt(m2);
        sh.thr = 2.5 * sigma;
      }
    }
    __syncthreads();
    double cnt[1] = {0.0};
    for (int m = threadIdx.x; m < M; m += kThreads) {
      const bool k = rbuf[m] <= sh.thr;
      keep[m] = k;
      cnt[0] += k;
    }
    block_sum<1>(cnt, sh.red);
    if (cnt[0] < 8.0) {
      // the max(8, M // 2) smallest residuals (ties: lowest index first)
      const int K = max(8, M / 2);
      if (w == 0) {
        const double v = warp_kth(rbuf, M, K - 1, sh.hist[0]);
        if (lane == 0) sh.thr = v;
      }
      __syncthreads();
      const double v = sh.thr;
      double lt[1] = {0.0};
      for (int m = threadIdx.x; m < M; m += kThreads) lt[0] += rbuf[m] < v;
      block_sum<1>(lt, sh.red);
      if (threadIdx.x == 0) {
        int need = K - (int)lt[0];
        for (int m = 0; m < M; ++m) {
          const bool less = rbuf[m] < v;
          const bool tie = rbuf[m] == v && need > 0;
          if (tie) --need;
          keep[m] = less || tie;
        }
      }
      __syncthreads();
    }
    fit_fundamental(p1, p2, keep, M, sh);
  } else {
    fit_fundamental(p1, p2, nullptr, M, sh);
  }

  // ---------------- _refit_on_inliers (ref/twoview.py:48-55)
  if (sh.status) {
    double F[9];
    for (int i = 0; i < 9; ++i) F[i] = sh.F[i];
    for (int m = threadIdx.x; m < M; m += kThreads) rbuf[m] = epi_abs(F, p1[m], p2[m]);
    __syncthreads();
    if (w == 0) {
      const double med = warp_median(rbuf, M, sh.hist[0]);
      if (lane == 0) sh.thr = fmax(10.0 * med, 1e-12);
    }
    __syncthreads();
    double cnt[1] = {0.0};
    for (int m = threadIdx.x; m < M; m += kThreads) {
      const bool k = rbuf[m] <= sh.thr;
      keep[m] = k;
      cnt[0] += k;
    }
    block_sum<1>(cnt, sh.red);
    if (cnt[0] >= 8.0 && cnt[0] < (double)M) fit_fundamental(p1, p2, keep, M, sh);
  }

  // ---------------- error sum (ref/distortion.py:121-122)
  if (!sh.status) {
    if (threadIdx.x == 0) {
      err_sum[job] = 0.0, n_err[job] = 0;
      if (F_out)
        for (int i = 0; i < 9; ++i) F_out[9 * job + i] = NAN;
    }
    return;
  }
  if (F_out && threadIdx.x < 9) F_out[9 * job + threadIdx.x] = sh.F[threadIdx.x];
  double F[9];
  for (int i = 0; i < 9; ++i) F[i] = sh.F[i];
  double e[1] = {0.0};
  for (int m = threadIdx.x; m < M; m += kThreads) e[0] += epi_abs(F, p1[m], p2[m]);
  block_sum<1>(e, sh.red);
  if (threadIdx.x == 0) err_sum[job] = e[0], n_err[job] = M;
}


// ======================================================================
// Robust homography fit (ref/twoview.py:136-201): the same job layout; the
// LMedS samples are 64 sequential 4-point draws (table from the host),
// a sample whose fit is degenerate is skipped, the score is the median
// Euclidean transfer error (non-finite -> inf), and the fits keep the
// reference's det / norm checks and positive-trace sign.
// ======================================================================

// transfer error ||proj(H x1) - x2|| (ref/twoview.py:126-134)
__device__ __forceinline__ double transfer_err(const double (&H)[9], double2 a, double2 b) {
  const double px = H[0] * a.x + H[1] * a.y + H[2];
  const double py = H[3] * a.x + H[4] * a.y + H[5];
  const double pz = H[6] * a.x + H[7] * a.y + H[8];
  const double dx = px / pz - b.x, dy = py / pz - b.y;
  if (!isfinite(dx) || !isfinite(dy)) return INFINITY;
  return sqrt(dx * dx + dy * dy);
}

// A rows of the normalised DLT (ref/twoview.py:186-190), accumulated into
// the 45 upper-triangle entries of A^T A
__device__ __forceinline__ void homog_rows(const Hartley& T, double2 a, double2 b, double (&n45)[45]) {
  const double x1[3] = {T.s1 * (a.x - T.cx1), T.s1 * (a.y - T.cy1), 1.0};
  const double x2x = T.s2 * (b.x - T.cx2), x2y = T.s2 * (b.y - T.cy2);
  double r0[9] = {0, 0, 0, -x1[0], -x1[1], -x1[2], x2y * x1[0], x2y * x1[1], x2y * x1[2]};
  double r1[9] = {x1[0], x1[1], x1[2], 0, 0, 0, -x2x * x1[0], -x2x * x1[1], -x2x * x1[2]};
  int q = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = i; j < 9; ++j) n45[q++] += r0[i] * r0[j] + r1[i] * r1[j];
}

// H from the normal matrix: smallest eigenvector, H = inv(T2) H T1, the
// degeneracy test on the unnormalised H, then Frobenius norm and trace sign.
// Returns false when degenerate (ref/twoview.py:191-200).
__device__ bool homog_from_normal(const double (&n45)[45], const Hartley& T, double (&H)[9]) {
  double a[9][9];
  int q = 0;
  for (int i = 0; i < 9; ++i)
    for (int j = i; j < 9; ++j) a[i][j] = a[j][i] = n45[q++];
  double h[9];
  smallest_eigvec9(a, h);
  // inv(T2) = [[1/s2, 0, cx2], [0, 1/s2, cy2], [0, 0, 1]]
  const double t1[9] = {T.s1, 0.0, -T.s1 * T.cx1, 0.0, T.s1, -T.s1 * T.cy1, 0.0, 0.0, 1.0};
  const double i2[9] = {1.0 / T.s2, 0.0, T.cx2, 0.0, 1.0 / T.s2, T.cy2, 0.0, 0.0, 1.0};
  double g[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += h[i * 3 + k] * t1[k * 3 + j];
      g[i * 3 + j] = acc;
    }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += i2[i * 3 + k] * g[k * 3 + j];
      H[i * 3 + j] = acc;
    }
  double nrm = 0.0;
  for (int i = 0; i < 9; ++i) nrm += H[i] * H[i];
  nrm = sqrt(nrm);
  const double det = H[0] * (H[4] * H[8] - H[5] * H[7]) - H[1] * (H[3] * H[8] - H[5] * H[6]) +
                     H[2] * (H[3] * H[7] - H[4] * H[6]);
  if (!(nrm >= 1e-15) || !(fabs(det) >= 1e-12)) return false;
  const double sg = (H[0] + H[4] + H[8]) / nrm < 0 ? -1.0 : 1.0;
  for (int i = 0; i < 9; ++i) H[i] = sg * (H[i] / nrm);
  return true;
}

// block-level least-squares homography on the masked points -> sh.F / sh.status
__device__ void fit_homography_block(const double2* p1, const double2* p2, const unsigned char* keep,
                                     int M, Shared& sh) {
  hartley(p1, p2, keep, M, sh);
  const Hartley T = sh.T;
  double n45[45];
#pragma unroll
  for (int i = 0; i < 45; ++i) n45[i] = 0.0;
  for (int m = threadIdx.x; m < M; m += kThreads) {
    if (keep && !keep[m]) continue;
    homog_rows(T, p1[m], p2[m], n45);
  }
  block_sum<45>(n45, sh.red);
  if (threadIdx.x == 0) {
    double H[9];
    if (homog_from_normal(n45, T, H))
      for (int i = 0; i < 9; ++i) sh.F[i] = H[i];
    else
      sh.status = 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads)
homog_fit_kernel(const int64_t* __restrict__ job_off, const double2* __restrict__ p1all,
                 const double2* __restrict__ p2all, const int32_t* __restrict__ sample_idx,
                 const int64_t* __restrict__ sample_off, double* __restrict__ H_out,
                 double* __restrict__ rbuf_all, unsigned char* __restrict__ keep_all) {
  __shared__ Shared sh;
  const int64_t job = blockIdx.x;
  const int64_t off = job_off[job];
  const int M = (int)(job_off[job + 1] - off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (M < 4) {
    if (threadIdx.x < 9) H_out[9 * job + threadIdx.x] = NAN;
    return;
  }
  const double2* p1 = p1all + off;
  const double2* p2 = p2all + off;
  double* rbuf = rbuf_all + kWarps * off;
  unsigned char* keep = keep_all + off;
  if (threadIdx.x == 0) sh.status = 1;
  __syncthreads();

  if (sample_off[job] >= 0) {
    // ---------------- LMedS (ref/twoview.py:156-177)
    if (threadIdx.x < kSamples) {
      const int32_t* idx = sample_idx + sample_off[job] + 4 * threadIdx.x;
      double2 a[4], b[4];
      for (int r = 0; r < 4; ++r) a[r] = p1[idx[r]], b[r] = p2[idx[r]];
      // Hartley normalisation of the 4 points (same expressions as hartley())
      double sx1 = 0, sy1 = 0, sx2 = 0, sy2 = 0;
      for (int r = 0; r < 4; ++r) sx1 += a[r].x, sy1 += a[r].y, sx2 += b[r].x, sy2 += b[r].y;
      Hartley T;
      T.cx1 = sx1 / 4.0, T.cy1 = sy1 / 4.0, T.cx2 = sx2 / 4.0, T.cy2 = sy2 / 4.0;
      double d1 = 0, d2 = 0;
      for (int r = 0; r < 4; ++r) {
        d1 += sqrt((a[r].x - T.cx1) * (a[r].x - T.cx1) + (a[r].y - T.cy1) * (a[r].y - T.cy1));
        d2 += sqrt((b[r].x - T.cx2) * (b[r].x - T.cx2) + (b[r].y - T.cy2) * (b[r].y - T.cy2));
      }
      T.s1 = sqrt(2.0) / fmax(d1 / 4.0, 1e-12);
      T.s2 = sqrt(2.0) / fmax(d2 / 4.0, 1e-12);
      double n45[45];
      for (int i = 0; i < 45; ++i) n45[i] = 0.0;
      for (int r = 0; r < 4; ++r) homog_rows(T, a[r], b[r], n45);
      double H[9];
      const bool ok = homog_from_normal(n45, T, H);
      for (int i = 0; i < 9; ++i) sh.Fk[threadIdx.x][i] = ok ? H[i] : NAN;
    }
    __syncthreads();
    double* mybuf = rbuf + (int64_t)w * M;
    for (int k = w; k < kSamples; k += kWarps) {
      double H[9];
      for (int i = 0; i < 9; ++i) H[i] = sh.Fk[k][i];
      if (isnan(H[0])) {  // degenerate sample: skipped (ref/twoview.py:162-165)
        if (lane == 0) sh.med[k] = NAN;
        continue;
      }
      for (int m = lane; m < M; m += 32) mybuf[m] = transfer_err(H, p1[m], p2[m]);
      __syncwarp();
      const double med = warp_median(mybuf, M, sh.hist[w]);
      if (lane == 0) sh.med[k] = med;
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int b = -1;
      double bm = INFINITY;
      for (int k = 0; k < kSamples; ++k)
        if (sh.med[k] < bm) bm = sh.med[k], b = k;  // strict <, from +inf (ref :166-167)
      sh.best = b;
    }
    __syncthreads();
    if (sh.best < 0) {
      fit_homography_block(p1, p2, nullptr, M, sh);
    } else {
      double H[9];
      for (int i = 0; i < 9; ++i) H[i] = sh.Fk[sh.best][i];
      for (int m = threadIdx.x; m < M; m += kThreads) rbuf[m] = transfer_err(H, p1[m], p2[m]);
      __syncthreads();
      if (w == 0) {
        double m2;
        if (M & 1) {
          const double x = warp_kth(rbuf, M, (M - 1) / 2, sh.hist[0]);
          m2 = x * x;
        } else {
          const double x = warp_kth(rbuf, M, M / 2 - 1, sh.hist[0]);
          const double y = warp_kth(rbuf, M, M / 2, sh.hist[0]);
          m2 = (x * x + y * y) / 2.0;
        }
        if (lane == 0) sh.thr = 2.5 * (1.4826 * (1.0 + 5.0 / max(M - 4, 1)) * sqrt(m2));
      }
      __syncthreads();
      double cnt[1] = {0.0};
      for (int m = threadIdx.x; m < M; m += kThreads) {
        const bool k = rbuf[m] <= sh.thr;
        keep[m] = k;
        cnt[0] += k;
      }
      block_sum<1>(cnt, sh.red);
      if (cnt[0] < 4.0) {
        const int K = max(4, M / 2);
        if (w == 0) {
          const double v = warp_kth(rbuf, M, K - 1, sh.hist[0]);
          if (lane == 0) sh.thr = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const double v = sh.thr;
          int lt = 0;
          for (int m = 0; m < M; ++m) lt += rbuf[m] < v;
          int need = K - lt;
          for (int m = 0; m < M; ++m) {
            const bool tie = rbuf[m] == v && need > 0;
            if (tie) --need;
            keep[m] = rbuf[m] < v || tie;
          }
        }
        __syncthreads();
      }
      fit_homography_block(p1, p2, keep, M, sh);
    }
  } else {
    fit_homography_block(p1, p2, nullptr, M, sh);
  }

  // ---------------- _refit_on_inliers (ref/twoview.py:48-55), min support 4
  if (sh.status) {
    double H[9];
    for (int i = 0; i < 9; ++i) H[i] = sh.F[i];
    for (int m = threadIdx.x; m < M; m += kThreads) rbuf[m] = transfer_err(H, p1[m], p2[m]);
    __syncthreads();
    if (w == 0) {
      const double med = warp_median(rbuf, M, sh.hist[0]);
      if (lane == 0) sh.thr = fmax(10.0 * med, 1e-12);
    }
    __syncthreads();
    double cnt[1] = {0.0};
    for (int m = threadIdx.x; m < M; m += kThreads) {
      const bool k = rbuf[m] <= sh.thr;
      keep[m] = k;
      cnt[0] += k;
    }
    block_sum<1>(cnt, sh.red);
    if (cnt[0] >= 4.0 && cnt[0] < (double)M) fit_homography_block(p1, p2, keep, M, sh);
  }
  if (threadIdx.x < 9) H_out[9 * job + threadIdx.x] = sh.status ? sh.F[threadIdx.x] : NAN;
}

}  // namespace
}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_fund_scratch_bytes(int64_t n_points) {
  if (n_points < 0) return 0;
  return (size_t)n_points * (kWarps * sizeof(double) + 1) + 256;
}

int fm_fund_score(int64_t n_jobs, const int64_t* job_off, const double* p1, const double* p2,
                  const int32_t* sample_idx, const int64_t* sample_off, double* err_sum,
                  int32_t* n_err, double* F_out, void* scratch, size_t scratch_bytes,
                  int64_t n_points, void* stream) {
  FM_REQUIRE(n_jobs >= 0 && n_points >= 0, "bad fundamental-fit sizes");
  if (n_jobs == 0) return FM_OK;
  FM_REQUIRE(job_off && p1 && p2 && sample_off && err_sum && n_err && scratch,
             "null fundamental-fit pointer");
  FM_REQUIRE(n_jobs <= 0x7fffffff, "too many fundamental-fit jobs");
  FM_REQUIRE(scratch_bytes >= fm_fund_scratch_bytes(n_points), "fundamental-fit scratch too small");
  double* rbuf = static_cast<double*>(scratch);
  unsigned char* keep = reinterpret_cast<unsigned char*>(rbuf + kWarps * n_points);
  fund_score_kernel<<<(unsigned)n_jobs, kThreads, 0, as_stream(stream)>>>(
      job_off, reinterpret_cast<const double2*>(p1), reinterpret_cast<const double2*>(p2),
      sample_idx, sample_off, err_sum, n_err, F_out, rbuf, keep);
  FM_LAUNCHED(fund_score_kernel);
  return FM_OK;
}

int fm_homog_fit(int64_t n_jobs, const int64_t* job_off, const double* p1, const double* p2,
                 const int32_t* sample_idx, const int64_t* sample_off, double* H_out,
                 void* scratch, size_t scratch_bytes, int64_t n_points, void* stream) {
  FM_REQUIRE(n_jobs >= 0 && n_points >= 0, "bad homography-fit sizes");
  if (n_jobs == 0) return FM_OK;
  FM_REQUIRE(job_off && p1 && p2 && sample_off && H_out && scratch, "null homography-fit pointer");
  FM_REQUIRE(n_jobs <= 0x7fffffff, "too many homography-fit jobs");
  FM_REQUIRE(scratch_bytes >= fm_fund_scratch_bytes(n_points), "homography-fit scratch too small");
  double* rbuf = static_cast<double*>(scratch);
  unsigned char* keep = reinterpret_cast<unsigned char*>(rbuf + kWarps * n_points);
  homog_fit_kernel<<<(unsigned)n_jobs, kThreads, 0, as_stream(stream)>>>(
      job_off, reinterpret_cast<const double2*>(p1), reinterpret_cast<const double2*>(p2),
      sample_idx, sample_off, H_out, rbuf, keep);
  FM_LAUNCHED(homog_fit_kernel);
  return FM_OK;
}

}  // extern "C"

// ======================================================================
// Focal voting (ref/focal.py:43-48, :81-120): votes[c] = sum over pairs p of
// exp((1 - s0/s1) / tau), s the singular values of E = K2^T F_p K1 with the
// candidate's K on the unknown side(s).  Block per candidate, thread per
// pair, fixed-order block sum; singular values by one-sided Jacobi (the
// column norms of E V).
// ======================================================================
namespace fm {
namespace {

__global__ void focal_votes_kernel(int32_t P, const double* __restrict__ F,
                                   const double* __restrict__ focal /* [C][P][2] */,
                                   const double* __restrict__ pp /* [P][4] cx1 cy1 cx2 cy2 */,
                                   double tau, double* __restrict__ votes) {
  __shared__ double red[kWarps];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int p = threadIdx.x; p < P; p += kThreads) {
    const double f1 = focal[(2 * (int64_t)c * P) + 2 * p], f2 = focal[(2 * (int64_t)c * P) + 2 * p + 1];
    const double K1[9] = {f1, 0.0, pp[4 * p], 0.0, f1, pp[4 * p + 1], 0.0, 0.0, 1.0};
    const double K2[9] = {f2, 0.0, pp[4 * p + 2], 0.0, f2, pp[4 * p + 3], 0.0, 0.0, 1.0};
    const double* Fp = F + 9 * (int64_t)p;
    double G[9], W[3][3];
    for (int i = 0; i < 3; ++i)  // G = F K1
      for (int l = 0; l < 3; ++l) {
        double s = 0.0;
        for (int k = 0; k < 3; ++k) s += Fp[i * 3 + k] * K1[k * 3 + l];
        G[i * 3 + l] = s;
      }
    for (int i = 0; i < 3; ++i)  // E = K2^T G
      for (int l = 0; l < 3; ++l) {
        double s = 0.0;
        for (int j = 0; j < 3; ++j) s += K2[j * 3 + i] * G[j * 3 + l];
        W[i][l] = s;
      }
    bool finite = true;
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l) finite &= isfinite(W[i][l]);
    double sv[3] = {NAN, NAN, NAN};
    if (finite) {
      for (int sweep = 0; sweep < 30; ++sweep) {
        bool rotated = false;
        for (int a = 0; a < 2; ++a)
          for (int b = a + 1; b < 3; ++b) {
            double al = 0.0, be = 0.0, ga = 0.0;
            for (int k = 0; k < 3; ++k) {
              al += W[k][a] * W[k][a];
              be += W[k][b] * W[k][b];
              ga += W[k][a] * W[k][b];
            }
            if (ga == 0.0 || fabs(ga) <= 1e-17 * sqrt(al * be)) continue;
            rotated = true;
            const double zeta = (be - al) / (2.0 * ga);
            const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
            for (int k = 0; k < 3; ++k) {
              const double wa = W[k][a], wb = W[k][b];
              W[k][a] = cs * wa - sn * wb;
              W[k][b] = sn * wa + cs * wb;
            }
          }
        if (!rotated) break;
      }
      for (int j = 0; j < 3; ++j) sv[j] = sqrt(W[0][j] * W[0][j] + W[1][j] * W[1][j] + W[2][j] * W[2][j]);
    }
    // s0 >= s1 >= s2
    double s0 = fmax(sv[0], fmax(sv[1], sv[2])), s2 = fmin(sv[0], fmin(sv[1], sv[2]));
    double s1 = sv[0] + sv[1] + sv[2] - s0 - s2;
    const double ratio = s0 / fmax(s1, 1e-300);
    acc += exp((1.0 - ratio) / tau);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0.0;
    for (int k = 0; k < kWarps; ++k) v += red[k];
    votes[c] = v;
  }
}

}  // namespace
}  // namespace fm

extern "C" int fm_focal_votes(int32_t n_cand, int32_t n_pairs, const double* F,
                              const double* focal, const double* principal, double tau,
                              double* votes_out, void* stream) {
  FM_REQUIRE(n_cand >= 0 && n_pairs >= 0 && tau > 0, "bad focal-vote arguments");
  if (n_cand == 0) return FM_OK;
  FM_REQUIRE(votes_out && (n_pairs == 0 || (F && focal && principal)), "null focal-vote pointer");
  fm::focal_votes_kernel<<<(unsigned)n_cand, fm::kThreads, 0, fm::as_stream(stream)>>>(
      n_pairs, F, focal, principal, tau, votes_out);
  FM_LAUNCHED(focal_votes_kernel);
  return FM_OK;
}
