// Relative-translation sphere search (SURVEY 8f "next" #1): the per-candidate
// mean epipolar error of ref/translation.py:52-55 and the cheirality counts of
// ref/twoview.py:246-253 that reestimate_relative (ref/translation.py:58-95)
// evaluates for every image pair of the pipeline.
//
// errors: one thread per candidate direction d; E = [d]_x R is formed once in
// registers and the pair's points stream through shared memory in tiles, so
// each (point, candidate) costs 12 fp64 FMAs (y = E x1, r = x2 . y) instead of
// the reference's 9-term products of a materialised (M, 9) term matrix.
// Deterministic: a fixed sequential order per candidate.
//
// depth counts: one thread per point pair; the DLT system A (4x4) of
// ref/twoview.py:220-243 is diagonalised by one-sided Jacobi rotations (the
// right singular vectors directly, no A^T A squaring), the singular vector of
// the smallest singular value is the homogeneous point, and the two depth
// signs are tested for both t and -t; a warp vote + one atomic per warp.
#include <cmath>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kTile = 256;  // points staged per tile

// blockIdx.y = pair k: points [off[k], off[k+1]), rotation R + 9k, candidates
// dirs + k * dir_stride (dir_stride 0: one lattice shared by all pairs),
// errors [k][C].
__global__ void sphere_errors_kernel(const double* __restrict__ x1, const double* __restrict__ x2,
                                     const int64_t* __restrict__ off, const double* __restrict__ Rs,
                                     const double* __restrict__ dirs, int64_t dir_stride, int C,
                                     double* __restrict__ errors) {
  __shared__ double sx1[kTile][3];
  __shared__ double sx2[kTile][3];
  const int k = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const double* R = Rs + 9 * (int64_t)k;
  const int64_t p0 = off[k], M = off[k + 1] - off[k];
  double E[9];
  {
    double d[3] = {0.0, 0.0, 1.0};
    const double* dk = dirs + k * dir_stride;
    if (c < C) d[0] = dk[3 * c], d[1] = dk[3 * c + 1], d[2] = dk[3 * c + 2];
    // [d]_x = [[0, -d2, d1], [d2, 0, -d0], [-d1, d0, 0]];  E = [d]_x R
    const double S[9] = {0.0, -d[2], d[1], d[2], 0.0, -d[0], -d[1], d[0], 0.0};
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int q = 0; q < 3; ++q)
        E[r * 3 + q] = S[r * 3 + 0] * R[0 * 3 + q] + S[r * 3 + 1] * R[1 * 3 + q] + S[r * 3 + 2] * R[2 * 3 + q];
  }
  double acc = 0.0;
  for (int64_t base = 0; base < M; base += kTile) {
    const int n = (int)(M - base < kTile ? M - base : kTile);
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * n; q += blockDim.x) {
      sx1[q / 3][q % 3] = x1[3 * (p0 + base) + q];
      sx2[q / 3][q % 3] = x2[3 * (p0 + base) + q];
    }
    __syncthreads();
    for (int m = 0; m < n; ++m) {
      const double a = sx1[m][0], b = sx1[m][1], w = sx1[m][2];
      const double y0 = fma(E[0], a, fma(E[1], b, E[2] * w));
      const double y1 = fma(E[3], a, fma(E[4], b, E[5] * w));
      const double y2 = fma(E[6], a, fma(E[7], b, E[8] * w));
      acc += fabs(fma(sx2[m][0], y0, fma(sx2[m][1], y1, sx2[m][2] * y2)));
    }
  }
  if (c < C) errors[(int64_t)k * C + c] = M > 0 ? acc / (double)M : 0.0;
}

// Right singular vector of the smallest singular value of a 4x4 matrix
// (one-sided Jacobi on the columns of A; A is destroyed).
__device__ void smallest_right_singular4(double (&A)[4][4], double (&v)[4]) {
  double V[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 30; ++sweep) {
    bool rotated = false;
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int q = p + 1; q < 4; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          al += A[k][p] * A[k][p];
          be += A[k][q] * A[k][q];
          ga += A[k][p] * A[k][q];
        }
        if (fabs(ga) <= 1e-15 * sqrt(al * be) || ga == 0.0) continue;
        rotated = true;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = cs * akp - sn * akq;
          A[k][q] = sn * akp + cs * akq;
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = cs * vkp - sn * vkq;
          V[k][q] = sn * vkp + cs * vkq;
        }
      }
    if (!rotated) break;
  }
  int best = 0;
  double bn = 1e308;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double nj = A[0][j] * A[0][j] + A[1][j] * A[1][j] + A[2][j] * A[2][j] + A[3][j] * A[3][j];
    if (nj < bn) {
      bn = nj;
      best = j;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = V[k][best];
}

// Camera 1 = [I | 0]; camera 2 = [R | t] (x2 ~ R x1 + t up to depth); c2 = -R^T t.
__device__ bool in_front(const double* R, const double* t, const double* c2, const double* x1,
                         const double* x2) {
  double A[4][4];
  // rows: x1x P1[2] - x1z P1[0], x1y P1[2] - x1z P1[1], same for camera 2
  const double P1[3][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}};
  const double P2[3][4] = {{R[0], R[1], R[2], t[0]}, {R[3], R[4], R[5], t[1]}, {R[6], R[7], R[8], t[2]}};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    A[0][k] = x1[0] * P1[2][k] - x1[2] * P1[0][k];
    A[1][k] = x1[1] * P1[2][k] - x1[2] * P1[1][k];
    A[2][k] = x2[0] * P2[2][k] - x2[2] * P2[0][k];
    A[3][k] = x2[1] * P2[2][k] - x2[2] * P2[1][k];
  }
  double X[4];
  smallest_right_singular4(A, X);
  double w = X[3];
  if (fabs(w) < 1e-15) w = 1e-15;  // ref/twoview.py:241
  const double p[3] = {X[0] / w, X[1] / w, X[2] / w};
  const double z1 = p[2];
  const double z2 = (p[0] - c2[0]) * R[6] + (p[1] - c2[1]) * R[7] + (p[2] - c2[2]) * R[8];
  return z1 > 0 && z2 > 0;
}

// blockIdx.y = pair k: the first min(M_k, cap) points, rotation Rs + 9k,
// translation ts + 3k; counts [k][2] for (t, -t).
__global__ void depth_counts_kernel(const double* __restrict__ Rs, const double* __restrict__ ts,
                                    const double* __restrict__ x1, const double* __restrict__ x2,
                                    const int64_t* __restrict__ off, int64_t cap,
                                    int32_t* __restrict__ counts) {
  const int k = blockIdx.y;
  const int64_t M = min(off[k + 1] - off[k], cap), p0 = off[k];
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double Rr[9], tp[3], tn[3], cp[3], cn[3];
#pragma unroll
  for (int q = 0; q < 9; ++q) Rr[q] = Rs[9 * (int64_t)k + q];
#pragma unroll
  for (int q = 0; q < 3; ++q) tp[q] = ts[3 * (int64_t)k + q], tn[q] = -tp[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) {  // c2 = -R^T t
    cp[q] = -(Rr[0 * 3 + q] * tp[0] + Rr[1 * 3 + q] * tp[1] + Rr[2 * 3 + q] * tp[2]);
    cn[q] = -cp[q];
  }
  bool fp = false, fn = false;
  if (m < M) {
    const double a[3] = {x1[3 * (p0 + m)], x1[3 * (p0 + m) + 1], x1[3 * (p0 + m) + 2]};
    const double b[3] = {x2[3 * (p0 + m)], x2[3 * (p0 + m) + 1], x2[3 * (p0 + m) + 2]};
    fp = in_front(Rr, tp, cp, a, b);
    fn = in_front(Rr, tn, cn, a, b);
  }
  const unsigned vp = __ballot_sync(0xffffffffu, fp), vn = __ballot_sync(0xffffffffu, fn);
  if ((threadIdx.x & 31) == 0) {
    if (vp) atomicAdd(counts + 2 * k, __popc(vp));
    if (vn) atomicAdd(counts + 2 * k + 1, __popc(vn));
  }
}

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

int fm_sphere_errors(const double* x1, const double* x2, int64_t M, const double* R,
                     const double* dirs, int32_t C, double* errors_out, void* stream) {
  FM_REQUIRE(M > 0 && C >= 0, "bad sphere-search sizes (M=%lld, C=%d)", (long long)M, C);
  FM_REQUIRE(x1 && x2 && R && (dirs || !C) && (errors_out || !C), "null sphere-search pointer");
  if (C == 0) return FM_OK;
  // one pair: offsets {0, M} in a tiny device scratch of the stream
  int64_t* off = nullptr;
  cudaStream_t st = as_stream(stream);
  FM_CUDA(cudaMallocAsync(&off, 2 * sizeof(int64_t), st));
  const int64_t h[2] = {0, M};
  FM_CUDA(cudaMemcpyAsync(off, h, sizeof(h), cudaMemcpyHostToDevice, st));
  sphere_errors_kernel<<<dim3((unsigned)ceil_div(C, 128), 1), 128, 0, st>>>(x1, x2, off, R, dirs, 0, C,
                                                                            errors_out);
  const cudaError_t le = cudaGetLastError();
  FM_CUDA(cudaFreeAsync(off, st));
  if (le != cudaSuccess) return cuda_fail(le, "sphere_errors_kernel", __FILE__, __LINE__);
  return FM_OK;
}

int fm_sphere_errors_batch(const double* x1, const double* x2, const int64_t* pair_off,
                           int32_t n_pairs, const double* R, const double* dirs,
                           int64_t dir_stride, int32_t C, double* errors_out, void* stream) {
  FM_REQUIRE(n_pairs >= 0 && C >= 0 && dir_stride >= 0, "bad batched sphere-search sizes");
  if (n_pairs == 0 || C == 0) return FM_OK;
  FM_REQUIRE(x1 && x2 && pair_off && R && dirs && errors_out, "null sphere-search pointer");
  FM_REQUIRE(n_pairs <= 65535, "at most 65535 pairs per batch");
  sphere_errors_kernel<<<dim3((unsigned)ceil_div(C, 128), (unsigned)n_pairs), 128, 0, as_stream(stream)>>>(
      x1, x2, pair_off, R, dirs, dir_stride, C, errors_out);
  FM_LAUNCHED(sphere_errors_kernel);
  return FM_OK;
}

int fm_depth_counts(const double* R, const double* t, const double* x1, const double* x2,
                    int64_t M, int32_t* counts_out, void* stream) {
  FM_REQUIRE(M >= 0 && R && t && counts_out, "bad depth-count arguments");
  cudaStream_t st = as_stream(stream);
  FM_CUDA(cudaMemsetAsync(counts_out, 0, 2 * sizeof(int32_t), st));
  if (M == 0) return FM_OK;
  FM_REQUIRE(x1 && x2, "null depth-count points");
  int64_t* off = nullptr;
  FM_CUDA(cudaMallocAsync(&off, 2 * sizeof(int64_t), st));
  const int64_t h[2] = {0, M};
  FM_CUDA(cudaMemcpyAsync(off, h, sizeof(h), cudaMemcpyHostToDevice, st));
  depth_counts_kernel<<<dim3((unsigned)ceil_div(M, 128), 1), 128, 0, st>>>(R, t, x1, x2, off, M, counts_out);
  const cudaError_t le = cudaGetLastError();
  FM_CUDA(cudaFreeAsync(off, st));
  if (le != cudaSuccess) return cuda_fail(le, "depth_counts_kernel", __FILE__, __LINE__);
  return FM_OK;
}

int fm_depth_counts_batch(const double* R, const double* t, const double* x1, const double* x2,
                          const int64_t* pair_off, int32_t n_pairs, int64_t max_points,
                          int32_t* counts_out, void* stream) {
  FM_REQUIRE(n_pairs >= 0 && max_points >= 0 && counts_out, "bad batched depth-count arguments");
  cudaStream_t st = as_stream(stream);
  if (n_pairs == 0) return FM_OK;
  FM_REQUIRE(R && t && x1 && x2 && pair_off, "null depth-count pointer");
  FM_REQUIRE(n_pairs <= 65535, "at most 65535 pairs per batch");
  FM_CUDA(cudaMemsetAsync(counts_out, 0, 2 * sizeof(int32_t) * (size_t)n_pairs, st));
  if (max_points == 0) return FM_OK;
  depth_counts_kernel<<<dim3((unsigned)ceil_div(max_points, 128), (unsigned)n_pairs), 128, 0, st>>>(
      R, t, x1, x2, pair_off, max_points, counts_out);
  FM_LAUNCHED(depth_counts_kernel);
  return FM_OK;
}

}  // extern "C"
