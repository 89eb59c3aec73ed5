// Library plumbing (error reporting, device query) and the small per-image
// kernels of the C ABI: rot6d maps, SO(3) projection, compose_essential and
// the flat Adam step.
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "fm_common.cuh"

namespace fm {

static thread_local char g_err[1024] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  return set_error(FM_ERR_CUDA, "CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                   cudaGetErrorString(e), what, file, line);
}

int sm_count() {
  static int cached = 0;
  if (cached) return cached;
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  cached = n > 0 ? n : 148;
  return cached;
}

// ------------------------------------------------------------ SO(3) projection
__device__ static void jacobi_sym3(double* A, double* V) {
  // Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (row-major A,
  // destroyed; eigenvalues end on the diagonal); V gets eigenvectors as columns.
  for (int k = 0; k < 9; ++k) V[k] = (k % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = A[1] * A[1] + A[2] * A[2] + A[5] * A[5];
    if (off < 1e-300) break;
    const int ps[3] = {0, 0, 1}, qs[3] = {1, 2, 2};
    for (int r = 0; r < 3; ++r) {
      const int p = ps[r], q = qs[r];
      const double apq = A[p * 3 + q];
      if (apq == 0.0) continue;
      const double theta = (A[q * 3 + q] - A[p * 3 + p]) / (2.0 * apq);
      const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
      for (int k = 0; k < 3; ++k) {  // A <- A J (columns p, q)
        const double akp = A[k * 3 + p], akq = A[k * 3 + q];
        A[k * 3 + p] = c * akp - s * akq;
        A[k * 3 + q] = s * akp + c * akq;
      }
      for (int k = 0; k < 3; ++k) {  // A <- J^T A (rows p, q)
        const double apk = A[p * 3 + k], aqk = A[q * 3 + k];
        A[p * 3 + k] = c * apk - s * aqk;
        A[q * 3 + k] = s * apk + c * aqk;
      }
      for (int k = 0; k < 3; ++k) {
        const double vkp = V[k * 3 + p], vkq = V[k * 3 + q];
        V[k * 3 + p] = c * vkp - s * vkq;
        V[k * 3 + q] = s * vkp + c * vkq;
      }
    }
  }
}

__device__ static double det3(const double* M) {
  return M[0] * (M[4] * M[8] - M[5] * M[7]) - M[1] * (M[3] * M[8] - M[5] * M[6]) +
         M[2] * (M[3] * M[7] - M[4] * M[6]);
}

__device__ void project_so3_dev(const double* M, double* R) {
  // Orthogonal polar factor Q of M by scaled Newton iteration, then the
  // reference's determinant fix U diag(1,1,sign det(UV^T)) V^T, which for
  // det(M) < 0 reflects Q across the smallest right singular vector.
  double X[9];
  for (int k = 0; k < 9; ++k) X[k] = M[k];
  const double d0 = det3(X);
  if (!(fabs(d0) > 1e-300) || !isfinite(d0)) {
    for (int k = 0; k < 9; ++k) R[k] = (k % 4 == 0) ? 1.0 : (isfinite(d0) ? 0.0 : NAN);
    return;
  }
  for (int it = 0; it < 60; ++it) {
    const double d = det3(X);
    // inverse transpose = cofactor / det
    double C[9];
    C[0] = (X[4] * X[8] - X[5] * X[7]) / d;
    C[1] = -(X[3] * X[8] - X[5] * X[6]) / d;
    C[2] = (X[3] * X[7] - X[4] * X[6]) / d;
    C[3] = -(X[1] * X[8] - X[2] * X[7]) / d;
    C[4] = (X[0] * X[8] - X[2] * X[6]) / d;
    C[5] = -(X[0] * X[7] - X[1] * X[6]) / d;
    C[6] = (X[1] * X[5] - X[2] * X[4]) / d;
    C[7] = -(X[0] * X[5] - X[2] * X[3]) / d;
    C[8] = (X[0] * X[4] - X[1] * X[3]) / d;
    double nx = 0, nc = 0;
    for (int k = 0; k < 9; ++k) {
      nx += X[k] * X[k];
      nc += C[k] * C[k];
    }
    const double gamma = (it < 8) ? sqrt(sqrt(nc / nx)) : 1.0;
    double diff = 0;
    for (int k = 0; k < 9; ++k) {
      const double nxk = 0.5 * (gamma * X[k] + C[k] / gamma);
      diff += (nxk - X[k]) * (nxk - X[k]);
      X[k] = nxk;
    }
    if (diff < 1e-30 && it >= 1) break;
  }
  if (d0 > 0) {
    for (int k = 0; k < 9; ++k) R[k] = X[k];
    return;
  }
  // det < 0: H = Q^T M (symmetric positive definite); smallest eigenvector v3
  double H[9], V[9];
  mat3_mul_at(X, M, H);
  for (int r = 0; r < 3; ++r)
    for (int c = r + 1; c < 3; ++c) {
      const double s = 0.5 * (H[r * 3 + c] + H[c * 3 + r]);
      H[r * 3 + c] = s;
      H[c * 3 + r] = s;
    }
  jacobi_sym3(H, V);
  int kmin = 0;
  if (H[4] < H[kmin * 4]) kmin = 1;
  if (H[8] < H[kmin * 4]) kmin = 2;
  const double v[3] = {V[0 * 3 + kmin], V[1 * 3 + kmin], V[2 * 3 + kmin]};
  // R = Q (I - 2 v v^T)
  for (int r = 0; r < 3; ++r) {
    const double qv = X[r * 3 + 0] * v[0] + X[r * 3 + 1] * v[1] + X[r * 3 + 2] * v[2];
    for (int c = 0; c < 3; ++c) R[r * 3 + c] = X[r * 3 + c] - 2.0 * qv * v[c];
  }
}

// ----------------------------------------------------------------- kernels
__global__ void rot6d_to_matrix_kernel(const double* __restrict__ v6, int64_t n, int project,
                                       double* __restrict__ R, int32_t* flag) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double Rk[9];
  const int code = rot6d_to_R(v6 + 6 * k, Rk);
  if (code) {
    raise_flag(flag, code);
    for (int q = 0; q < 9; ++q) R[9 * k + q] = NAN;
    return;
  }
  if (project) {
    double P[9];
    project_so3_dev(Rk, P);
    for (int q = 0; q < 9; ++q) R[9 * k + q] = P[q];
  } else {
    for (int q = 0; q < 9; ++q) R[9 * k + q] = Rk[q];
  }
}

__global__ void rot6d_jacobian_kernel(const double* __restrict__ v6, int64_t n,
                                      double* __restrict__ J) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double Jk[54];
  rot6d_jacobian_dev(v6 + 6 * k, Jk);
  for (int q = 0; q < 54; ++q) J[54 * k + q] = Jk[q];
}

__global__ void project_so3_kernel(const double* __restrict__ M, int64_t n, double* __restrict__ R) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double Mk[9], Rk[9];
  for (int q = 0; q < 9; ++q) Mk[q] = M[9 * k + q];
  project_so3_dev(Mk, Rk);
  for (int q = 0; q < 9; ++q) R[9 * k + q] = Rk[q];
}

__global__ void compose_essential_kernel(const double* __restrict__ Ri, const double* __restrict__ Rj,
                                         const double* __restrict__ oi, const double* __restrict__ oj,
                                         int64_t n, double* __restrict__ E) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  double a[9], b[9], dc[3], t[3], Rrel[9], Ek[9];
  for (int q = 0; q < 9; ++q) {
    a[q] = Ri[9 * k + q];
    b[q] = Rj[9 * k + q];
  }
  essential(a, b, oi + 3 * k, oj + 3 * k, dc, t, Rrel, Ek);
  for (int q = 0; q < 9; ++q) E[9 * k + q] = Ek[q];
}

// Adam with bias correction (ref/optim.py:24-36).  The non-finite check of
// ref/optim.py:28-29 runs over the whole gradient before any update: pass 1
// flags, pass 2 (same launch, after a grid-wide condition) is replaced by a
// per-element guard -- every element whose gradient vector is non-finite
// stops the whole update because the flag is checked by the host before the
// parameters are used (the step is then discarded with the exception).
__global__ void adam_check_kernel(const double* __restrict__ g, int64_t n, int32_t* flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(g[k])) raise_flag(flag, FM_ERR_NONFINITE_GRAD);
}

__global__ void adam_update_kernel(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                                   const double* __restrict__ g, int64_t n, double lr, double b1,
                                   double b2, double eps, double bc1, double bc2, const int32_t* flag) {
  if (flag && *flag) return;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    // explicit _rn intrinsics: no FMA contraction, so the update rounds
    // exactly like the numpy expression of ref/optim.py:33-35
    const double gk = g[k];
    const double mk = __dadd_rn(__dmul_rn(b1, m[k]), __dmul_rn(1.0 - b1, gk));
    const double vk = __dadd_rn(__dmul_rn(b2, v[k]), __dmul_rn(1.0 - b2, __dmul_rn(gk, gk)));
    m[k] = mk;
    v[k] = vk;
    p[k] = __dsub_rn(p[k], __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, bc1)),
                                     __dadd_rn(sqrt(__ddiv_rn(vk, bc2)), eps)));
  }
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_abi_version(void) { return FM_ABI_VERSION; }

const char* fm_last_error(void) { return g_err; }

int fm_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int fm_rot6d_to_matrix(const double* rot6d, int64_t n, int32_t project, double* R_out,
                       int32_t* flag, void* stream) {
  FM_REQUIRE(n >= 0, "negative count");
  if (n == 0) return FM_OK;
  rot6d_to_matrix_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      rot6d, n, project, R_out, flag);
  FM_LAUNCHED(rot6d_to_matrix_kernel);
  return FM_OK;
}

int fm_rot6d_jacobian(const double* rot6d, int64_t n, double* J_out, void* stream) {
  FM_REQUIRE(n >= 0, "negative count");
  if (n == 0) return FM_OK;
  rot6d_jacobian_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(rot6d, n, J_out);
  FM_LAUNCHED(rot6d_jacobian_kernel);
  return FM_OK;
}

int fm_project_to_so3(const double* M, int64_t n, double* R_out, void* stream) {
  FM_REQUIRE(n >= 0, "negative count");
  if (n == 0) return FM_OK;
  project_so3_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(M, n, R_out);
  FM_LAUNCHED(project_so3_kernel);
  return FM_OK;
}

int fm_compose_essential(const double* R_i, const double* R_j, const double* o_i,
                         const double* o_j, int64_t n, double* E_out, void* stream) {
  FM_REQUIRE(n >= 0, "negative count");
  if (n == 0) return FM_OK;
  compose_essential_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      R_i, R_j, o_i, o_j, n, E_out);
  FM_LAUNCHED(compose_essential_kernel);
  return FM_OK;
}

int fm_adam_step(double* params, double* adam_m, double* adam_v, const double* grad, int64_t n,
                 int64_t t, double lr, double beta1, double beta2, double eps, int32_t* flag,
                 void* stream) {
  FM_REQUIRE(n >= 0 && t >= 1, "bad Adam step arguments (n=%lld, t=%lld)", (long long)n,
             (long long)t);
  if (n == 0) return FM_OK;
  const int blocks = (int)std::min<int64_t>(ceil_div(n, 256), 4 * sm_count());
  cudaStream_t s = as_stream(stream);
  adam_check_kernel<<<blocks, 256, 0, s>>>(grad, n, flag);
  FM_LAUNCHED(adam_check_kernel);
  const double bc1 = 1.0 - pow(beta1, (double)t);
  const double bc2 = 1.0 - pow(beta2, (double)t);
  adam_update_kernel<<<blocks, 256, 0, s>>>(params, adam_m, adam_v, grad, n, lr, beta1, beta2, eps,
                                            bc1, bc2, flag);
  FM_LAUNCHED(adam_update_kernel);
  return FM_OK;
}

}  // extern "C"
