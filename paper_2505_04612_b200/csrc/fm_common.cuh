// Shared device helpers of the FastMap B200 hot path.
//
// Geometry follows the reference exactly (file:line cited per function); the
// arithmetic is fp64 everywhere except the point-pair moment accumulation
// (see fm_point_pass.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/fastmap_b200.h"

namespace fm {

// ---------------------------------------------------------------- host side
int set_error(int code, const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define FM_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e__ = (call);                                                \
    if (e__ != cudaSuccess)                                                  \
      return ::fm::cuda_fail(e__, #call, __FILE__, __LINE__);                \
  } while (0)

#define FM_LAUNCHED(name) FM_CUDA(cudaGetLastError())

#define FM_REQUIRE(cond, ...)                                                \
  do {                                                                       \
    if (!(cond)) return ::fm::set_error(FM_ERR_INVALID, __VA_ARGS__);        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Bump allocator over caller-provided scratch (256-byte aligned pieces).
struct Scratch {
  char* base;
  size_t cap;
  size_t used;
  Scratch(void* p, size_t n) : base(static_cast<char*>(p)), cap(n), used(0) {}
  template <typename T>
  T* take(size_t count) {
    size_t off = (used + 255) & ~size_t(255);
    used = off + count * sizeof(T);
    return reinterpret_cast<T*>(base + off);
  }
  bool ok() const { return used <= cap; }
};
inline size_t scratch_round(size_t bytes) { return (bytes + 255) & ~size_t(255); }

int sm_count();

// Sum all-reduce of n doubles in place over an NCCL communicator (comm NULL:
// one rank, no-op); stream-ordered, CUDA-graph capturable (fm_dist.cu).
int nccl_allreduce_sum_f64(double* buf, size_t n, void* comm, cudaStream_t st);

// -------------------------------------------------------------- device side
__device__ __forceinline__ void raise_flag(int32_t* flag, int code) {
  if (flag) atomicCAS(flag, 0, code);
}

__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// 6D -> rotation matrix by Gram-Schmidt (ref/optim.py:39-59).  Columns are
// b1, b2, b1 x b2; R is row-major.  Returns 0 or the degeneracy code.
__device__ __forceinline__ int rot6d_to_R(const double* v, double* R) {
  const double a0 = v[0], a1 = v[1], a2 = v[2];
  const double b0 = v[3], b1 = v[4], b2 = v[5];
  const double na = sqrt(a0 * a0 + a1 * a1 + a2 * a2);
  if (na < 1e-12) return FM_ERR_ROT6D_ZERO;
  const double e0 = a0 / na, e1 = a1 / na, e2 = a2 / na;
  const double d = e0 * b0 + e1 * b1 + e2 * b2;
  const double u0 = b0 - d * e0, u1 = b1 - d * e1, u2 = b2 - d * e2;
  const double nu = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
  if (nu < 1e-12) return FM_ERR_ROT6D_COLLINEAR;
  const double f0 = u0 / nu, f1 = u1 / nu, f2 = u2 / nu;
  R[0] = e0; R[1] = f0; R[2] = e1 * f2 - e2 * f1;
  R[3] = e1; R[4] = f1; R[5] = e2 * f0 - e0 * f2;
  R[6] = e2; R[7] = f2; R[8] = e0 * f1 - e1 * f0;
  return 0;
}

// Vector-Jacobian product of rot6d_to_R: g6 = J^T vec(gR), where J is the
// (9, 6) Jacobian of ref/optim.py:68-110.  Back-propagates through the
// Gram-Schmidt steps instead of forming J (so it is not the reference's
// arithmetic anyway): one reciprocal per norm and products instead of twelve
// serial divisions on the Adam step's critical path (within ~1 ulp).
__device__ __forceinline__ void rot6d_vjp(const double* v, const double* gR, double* g6) {
  const double a[3] = {v[0], v[1], v[2]};
  const double b[3] = {v[3], v[4], v[5]};
  const double na = sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
  const double ina = 1.0 / na;
  double e[3] = {a[0] * ina, a[1] * ina, a[2] * ina};
  const double d = e[0] * b[0] + e[1] * b[1] + e[2] * b[2];
  double u[3] = {b[0] - d * e[0], b[1] - d * e[1], b[2] - d * e[2]};
  const double nu = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
  const double inu = 1.0 / nu;
  double f[3] = {u[0] * inu, u[1] * inu, u[2] * inu};
  double ge[3] = {gR[0], gR[3], gR[6]};
  double gf[3] = {gR[1], gR[4], gR[7]};
  const double gh[3] = {gR[2], gR[5], gR[8]};
  // h = e x f  ->  ge += f x gh ; gf += gh x e
  ge[0] += f[1] * gh[2] - f[2] * gh[1];
  ge[1] += f[2] * gh[0] - f[0] * gh[2];
  ge[2] += f[0] * gh[1] - f[1] * gh[0];
  gf[0] += gh[1] * e[2] - gh[2] * e[1];
  gf[1] += gh[2] * e[0] - gh[0] * e[2];
  gf[2] += gh[0] * e[1] - gh[1] * e[0];
  // f = u / |u|
  const double fg = f[0] * gf[0] + f[1] * gf[1] + f[2] * gf[2];
  double gu[3];
  for (int k = 0; k < 3; ++k) gu[k] = (gf[k] - f[k] * fg) * inu;
  // u = b - (e.b) e
  const double eg = e[0] * gu[0] + e[1] * gu[1] + e[2] * gu[2];
  for (int k = 0; k < 3; ++k) {
    g6[3 + k] = gu[k] - e[k] * eg;
    ge[k] += -eg * b[k] - d * gu[k];
  }
  // e = a / |a|
  const double ee = e[0] * ge[0] + e[1] * ge[1] + e[2] * ge[2];
  for (int k = 0; k < 3; ++k) g6[k] = (ge[k] - e[k] * ee) * ina;
}

// Full Jacobian (9 x 6, row-major flat R rows) -- only for the API function
// rot6d_jacobian (ref/optim.py:68-110); built from 6 VJPs is wasteful, so we
// build it column-wise with forward-mode derivatives.
__device__ __forceinline__ void rot6d_jacobian_dev(const double* v, double* J) {
  for (int row = 0; row < 9; ++row) {
    double gR[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    gR[row] = 1.0;
    double g6[6];
    rot6d_vjp(v, gR, g6);
    for (int p = 0; p < 6; ++p) J[row * 6 + p] = g6[p];
  }
}

// Polar projection onto SO(3): the nearest rotation in Frobenius norm
// (ref/model.py:112-116 computes U diag(1,1,sign det(U V^T)) V^T by SVD).
// Newton iteration X <- (X + X^{-T}) / 2 converges to the orthogonal polar
// factor; a final sign fix handles det < 0 inputs the same way the SVD
// formula does (flip the direction of the smallest singular vector) by
// falling back to a Jacobi SVD for those rare inputs.
__device__ void project_so3_dev(const double* M, double* R);

// 3x3 helpers (row-major)
__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[r * 3 + c] = A[r * 3 + 0] * B[0 * 3 + c] + A[r * 3 + 1] * B[1 * 3 + c] +
                     A[r * 3 + 2] * B[2 * 3 + c];
}
// C = A B^T
__device__ __forceinline__ void mat3_mul_bt(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[r * 3 + c] = A[r * 3 + 0] * B[c * 3 + 0] + A[r * 3 + 1] * B[c * 3 + 1] +
                     A[r * 3 + 2] * B[c * 3 + 2];
}
// C = A^T B
__device__ __forceinline__ void mat3_mul_at(const double* A, const double* B, double* C) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      C[r * 3 + c] = A[0 * 3 + r] * B[0 * 3 + c] + A[1 * 3 + r] * B[1 * 3 + c] +
                     A[2 * 3 + r] * B[2 * 3 + c];
}

// Essential matrix from world-to-camera rotations and centres
// (ref/epipolar.py:62-70 and :112-117): t = -R_j (c_j - c_i),
// R_rel = R_j R_i^T, E = [t]x R_rel.
__device__ __forceinline__ void essential(const double* Ri, const double* Rj,
                                          const double* ci, const double* cj,
                                          double* dc, double* t, double* Rrel,
                                          double* E) {
  dc[0] = cj[0] - ci[0];
  dc[1] = cj[1] - ci[1];
  dc[2] = cj[2] - ci[2];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    t[r] = -(Rj[r * 3 + 0] * dc[0] + Rj[r * 3 + 1] * dc[1] + Rj[r * 3 + 2] * dc[2]);
  mat3_mul_bt(Rj, Ri, Rrel);
  // [t]x = [[0,-t2,t1],[t2,0,-t0],[-t1,t0,0]]
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    E[0 * 3 + c] = -t[2] * Rrel[1 * 3 + c] + t[1] * Rrel[2 * 3 + c];
    E[1 * 3 + c] = t[2] * Rrel[0 * 3 + c] - t[0] * Rrel[2 * 3 + c];
    E[2 * 3 + c] = -t[1] * Rrel[0 * 3 + c] + t[0] * Rrel[1 * 3 + c];
  }
}

// Symmetric index of an unordered pair (p, q) of {0,1,2}: 00,01,02,11,12,22.
__host__ __device__ __forceinline__ constexpr int sym3(int p, int q) {
  return p <= q ? (p == 0 ? q : (p == 1 ? 2 + q : 5)) : (q == 0 ? p : (q == 1 ? 2 + p : 5));
}

}  // namespace fm
