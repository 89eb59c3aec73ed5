// Image-pair level of the epipolar adjustment: per-pair Frobenius-normalised
// essential/fundamental matrices, the quadratic loss and its gradient in the
// packed [rot6d | centers | log_focal] parameters, deterministic per-image and
// per-camera reductions, and the fused Adam step loop
// (ref/epipolar.py:109-138, :172-248, :302-308; ref/optim.py:24-36).
//
// Per step: O(image pairs) work, independent of the number of point pairs
// (the paper's claim, ref/epipolar.py:3-7).  All fp64.  A step is
//   pair_grad   (thread / image pair)  -> per-pair dL/dR_i, dL/dR_j, dL/dc, dL/dphi
//   image_adam  (warp / image)         -> gather over the image's incidences in
//                                         fixed order, 6D VJP, Adam, new R
//   cam_chunk   (block / chunk)        -> fixed-order partial focal sums
//   cam_adam    (thread / camera)      -> focal gradient, Adam
// and is replayed from a CUDA graph in the hot loop.
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <cmath>
#include <cstring>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kPG = 24;          // per-pair gradient record: gRi 9, gRj 9, gdc 3, gphi_i, gphi_j, loss
constexpr int kMaxSteps = 4096;  // steps per fm_epi_adam_steps call (bias-correction table)
constexpr int kPairBlock = 64;   // pair_grad threads per block
// Focal gradients with few cameras: pair_grad sums each block's per-camera
// terms (a fixed tree) into cpart[c][block] and image_reduce reduces the
// block partials with a warp per camera -- no incidence gather, no ticket.
// More cameras: the per-camera incidence chunks (cam_chunk_*).
constexpr int kBlockCams = 8;
constexpr int kIncPad = 128;  // per-image padded incidence table (image_reduce's first batch)
__host__ __device__ inline bool cams_by_block(const fm_pair_graph& g) {
  return g.refine_focal && g.n_cameras > 0 && g.n_cameras <= kBlockCams;
}
inline int64_t pair_blocks(const fm_pair_graph& g) { return ceil_div(g.n_pairs, kPairBlock); }
inline size_t cpart_len(const fm_pair_graph& g) {
  size_t n = (size_t)std::max(g.n_cam_chunks, 1);
  if (cams_by_block(g)) n = std::max(n, (size_t)g.n_cameras * (size_t)pair_blocks(g));
  return n;
}

struct EpiScratch {
  double* R;      // [N][9] rotations, then [n_cameras] focal scales exp(-log_focal)
  double* pg;     // [kPG][P]
  double* cpart;  // [n_cam_chunks] or [n_cameras][pair blocks] (cams_by_block)
  double* lpart;  // [loss blocks]
  double* sched;  // [2 + 2*kMaxSteps + 1]: lr, scale, bc1[], bc2[], peer-step epoch
  unsigned int* ticket;  // camera-chunk completion counter (last block finalises)
  int* inc_pad;          // [N][kIncPad] first incidences per image, -1 padded
};

// image_reduce blocks of the camera role: a warp per camera (cams_by_block)
// or a block per incidence chunk.
inline int cam_role_blocks(const fm_pair_graph& g) {
  if (!(g.refine_focal && g.n_cameras > 0)) return 0;
  return cams_by_block(g) ? (int)ceil_div(g.n_cameras, 2) : g.n_cam_chunks;
}

int loss_blocks(int64_t P) { return (int)std::min<int64_t>(std::max<int64_t>(ceil_div(P, 1024), 1), 1024); }

size_t scratch_need(const fm_pair_graph& g) {
  size_t b = 0;
  b += scratch_round(((size_t)g.n_images * 9 + std::max(g.n_cameras, 1)) * sizeof(double));
  b += scratch_round((size_t)g.n_pairs * kPG * sizeof(double));
  b += scratch_round(cpart_len(g) * sizeof(double));
  b += scratch_round((size_t)loss_blocks(g.n_pairs) * sizeof(double));
  b += scratch_round((size_t)(3 + 2 * kMaxSteps) * sizeof(double));
  b += scratch_round(sizeof(unsigned int));
  b += scratch_round((size_t)std::max(g.n_images, 1) * kIncPad * sizeof(int));
  return b + 256;
}

bool carve(const fm_pair_graph& g, void* p, size_t n, EpiScratch& s) {
  Scratch sc(p, n);
  s.R = sc.take<double>((size_t)g.n_images * 9 + std::max(g.n_cameras, 1));
  s.pg = sc.take<double>((size_t)g.n_pairs * kPG);
  s.cpart = sc.take<double>(cpart_len(g));
  s.lpart = sc.take<double>((size_t)loss_blocks(g.n_pairs));
  s.sched = sc.take<double>((size_t)(3 + 2 * kMaxSteps));
  s.ticket = sc.take<unsigned int>(1);
  s.inc_pad = sc.take<int>((size_t)std::max(g.n_images, 1) * kIncPad);
  return p != nullptr && sc.ok();
}

// ------------------------------------------------------------------ kernels
// Per image: R from the 6D parameters; per camera (n_cam > 0 when focals
// are refined): the focal scale exp(-log_focal) after the rotations, so the
// pair kernels read it instead of evaluating two fp64 exps per pair.
__global__ void image_rot_kernel(const double* __restrict__ params, int n, double* __restrict__ R,
                                 int32_t* flag, int n_cam) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n_cam) R[9 * n + k] = exp(-params[9 * n + k]);
  if (k >= n) return;
  double Rk[9];
  const int code = rot6d_to_R(params + 6 * k, Rk);
  if (code) raise_flag(flag, code);
#pragma unroll
  for (int q = 0; q < 9; ++q) R[9 * k + q] = Rk[q];
}

int launch_image_rot(const fm_pair_graph& g, const double* params, double* R, int32_t* flag,
                     cudaStream_t st) {
  const int n_cam = g.refine_focal ? g.n_cameras : 0;
  const int n = std::max(g.n_images, n_cam);
  if (n == 0) return FM_OK;
  image_rot_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(params, g.n_images, R, flag, n_cam);
  FM_LAUNCHED(image_rot_kernel);
  return FM_OK;
}

// Forward geometry of one image pair (ref/epipolar.py:109-138).
struct PairFwd {
  double Ri[9], Rj[9], dc[3], t[3], Rrel[9], E[9], G[9], gh[9];
  double nrm, di, dj;
};

// EXACT: ghat = G / ||G|| by division, as the reference (the point passes'
// linearisation point, whose residuals decide pruning); otherwise one
// reciprocal and nine products (the per-step gradient path, <= 1.5 ulp).
// Where a step reads the per-image geometry: rotation of image i at
// R + rs * i, its centre at C + cs * i, camera c's focal scale exp(-log_focal)
// at F[c] (geo_split: R [N][9] | F from image_rot_kernel, the packed params'
// centres).
struct Geo {
  const double* R;
  const double* C;
  const double* F;
  int rs, cs;
};
__device__ __forceinline__ Geo geo_split(const fm_pair_graph& g, const double* params, const double* R) {
  return Geo{R, params + 6 * (int64_t)g.n_images, R + 9 * (int64_t)g.n_images, 9, 3};
}

template <bool EXACT>
__device__ __forceinline__ void pair_forward(const fm_pair_graph& g, const Geo& geo, int64_t n,
                                             PairFwd& f) {
  const int i = g.pair_i[n], j = g.pair_j[n];
#pragma unroll
  for (int q = 0; q < 9; ++q) {
    f.Ri[q] = geo.R[(int64_t)geo.rs * i + q];
    f.Rj[q] = geo.R[(int64_t)geo.rs * j + q];
  }
  const double* ci = geo.C + (int64_t)geo.cs * i;
  const double* cj = geo.C + (int64_t)geo.cs * j;
  essential(f.Ri, f.Rj, ci, cj, f.dc, f.t, f.Rrel, f.E);
  if (g.refine_focal) {
    f.di = geo.F[g.pair_ci[n]];  // exp(-log_focal), image_rot_kernel / cam_update
    f.dj = geo.F[g.pair_cj[n]];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b)
        f.G[a * 3 + b] = (a < 2 ? f.dj : 1.0) * f.E[a * 3 + b] * (b < 2 ? f.di : 1.0);
  } else {
    f.di = f.dj = 1.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) f.G[q] = f.E[q];
  }
  double ss = 0;
#pragma unroll
  for (int q = 0; q < 9; ++q) ss += f.G[q] * f.G[q];
  f.nrm = fmax(sqrt(ss), 1e-15);
  if (EXACT) {
#pragma unroll
    for (int q = 0; q < 9; ++q) f.gh[q] = f.G[q] / f.nrm;
  } else {
    const double inv = 1.0 / f.nrm;
#pragma unroll
    for (int q = 0; q < 9; ++q) f.gh[q] = f.G[q] * inv;
  }
}

__global__ void pair_ghat_kernel(const fm_pair_graph g, const double* __restrict__ params,
                                 const double* __restrict__ R, double* __restrict__ ghat) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n >= g.n_pairs) return;
  PairFwd f;
  pair_forward<true>(g, geo_split(g, params, R), n, f);
#pragma unroll
  for (int q = 0; q < 9; ++q) ghat[q * g.n_pairs + n] = f.gh[q];
}

// u = W x for the Kronecker-structured W given by 36 moments:
// (W x)[p][r] = sum_{q,s} mom[sym(p,q)][sym(r,s)] x[q][s]
template <typename T>
__device__ __forceinline__ void mom_apply(const T* __restrict__ mom, int64_t P, int64_t n,
                                          const double* x, double* u) {
  double m[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) m[k] = (double)mom[k * P + n];
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double acc = 0;
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int s = 0; s < 3; ++s) acc = fma(m[sym3(p, q) * 6 + sym3(r, s)], x[q * 3 + s], acc);
      u[p * 3 + r] = acc;
    }
}

// Loss term and full backward of one pair (ref/epipolar.py:172-232).
struct PairGradOut {
  double gRi[9], gRj[9], gdc[3], gphi_i, gphi_j, loss;
};

template <int KIND>
__device__ __forceinline__ void pair_grad_one(const fm_pair_graph& g, const fm_quad_model& q,
                                              const Geo& geo, const double scale, const int64_t n,
                                              PairGradOut& o) {
  const int64_t P = g.n_pairs;
  PairFwd f;
  pair_forward<false>(g, geo, n, f);

  double u[9], Ln;
  if (KIND == FM_QUAD_SHIFTED32) {
    // ghat^T W ghat = s0 + 2 d^T v + d^T W d, d = ghat - ghat0, v = W ghat0
    double d[9], Wd[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) d[k] = f.gh[k] - q.ghat0[k * P + n];
    mom_apply(q.mom32, P, n, d, Wd);
    double acc = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const double v = (double)q.vgrad[k * P + n];
      u[k] = v + Wd[k];
      acc = fma(d[k], v + u[k], acc);
    }
    Ln = q.s0[n] + acc;
  } else if (KIND == FM_QUAD_MOM64) {
    mom_apply(q.mom64, P, n, f.gh, u);
    Ln = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) Ln = fma(f.gh[k], u[k], Ln);
  } else {  // dense caller-given W (row-major 9x9)
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      double acc = 0;
#pragma unroll
      for (int l = 0; l < 9; ++l) acc = fma(q.w81[(k * 9 + l) * P + n], f.gh[l], acc);
      u[k] = acc;
    }
    Ln = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) Ln = fma(f.gh[k], u[k], Ln);
  }
  const double loss_n = scale * Ln;
  // d loss / d ghat = (2/Z) 2 W ghat, then through the normalisation
  double gg[9], dot = 0;
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    gg[k] = 2.0 * scale * u[k];
    dot = fma(f.gh[k], gg[k], dot);
  }
  double gG[9];
  const double inv_nrm = 1.0 / f.nrm;  // one division instead of nine (<= 1.5 ulp apart)
#pragma unroll
  for (int k = 0; k < 9; ++k) gG[k] = (gg[k] - f.gh[k] * dot) * inv_nrm;

  double gE[9], gphi_i = 0, gphi_j = 0;
  if (g.refine_focal) {
    double si = 0, sj = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double fa = a < 2 ? f.dj : 1.0, fb = b < 2 ? f.di : 1.0;
        gE[a * 3 + b] = fa * gG[a * 3 + b] * fb;
        if (b < 2) si += gG[a * 3 + b] * (fa * f.E[a * 3 + b]);  // (Dj E) columns 0,1
        if (a < 2) sj += gG[a * 3 + b] * (f.E[a * 3 + b] * fb);  // (E Di) rows 0,1
      }
    gphi_i = -f.di * si;
    gphi_j = -f.dj * sj;
  } else {
#pragma unroll
    for (int k = 0; k < 9; ++k) gE[k] = gG[k];
  }
  // E = [t]x R_rel:  M_rel = [t]x^T gE,  Pm = gE R_rel^T
  const double* t = f.t;
  double Mrel[9], Pm[9];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    // [t]x^T = [[0,t2,-t1],[-t2,0,t0],[t1,-t0,0]]
    Mrel[0 * 3 + c] = t[2] * gE[1 * 3 + c] - t[1] * gE[2 * 3 + c];
    Mrel[1 * 3 + c] = -t[2] * gE[0 * 3 + c] + t[0] * gE[2 * 3 + c];
    Mrel[2 * 3 + c] = t[1] * gE[0 * 3 + c] - t[0] * gE[1 * 3 + c];
  }
  mat3_mul_bt(gE, f.Rrel, Pm);
  const double gt[3] = {Pm[7] - Pm[5], Pm[2] - Pm[6], Pm[3] - Pm[1]};
  // t = -R_j dc
  double gdc[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) gdc[c] = -(f.Rj[0 * 3 + c] * gt[0] + f.Rj[1 * 3 + c] * gt[1] + f.Rj[2 * 3 + c] * gt[2]);
  double gRj[9], gRi[9];
  mat3_mul(Mrel, f.Ri, gRj);
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) gRj[a * 3 + b] -= gt[a] * f.dc[b];
  mat3_mul_at(Mrel, f.Rj, gRi);

#pragma unroll
  for (int k = 0; k < 9; ++k) {
    o.gRi[k] = gRi[k];
    o.gRj[k] = gRj[k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) o.gdc[k] = gdc[k];
  o.gphi_i = gphi_i;
  o.gphi_j = gphi_j;
  o.loss = loss_n;
}

// Step kernel: a thread per pair (pair_grad_one) + the block's focal partials.
template <int KIND>
__global__ void __launch_bounds__(kPairBlock)
pair_grad_kernel(const fm_pair_graph g, const fm_quad_model q, const double* __restrict__ params,
                 const double* __restrict__ R, const double* __restrict__ sched,
                 double* __restrict__ pg, double* __restrict__ cpart, int32_t* flag) {
  const int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t P = g.n_pairs;
  // No early exit on a raised flag: a flagged run's later steps compute
  // harmless values and image_reduce, which checks the flag before Adam,
  // leaves the parameters alone (the flag load stays off this kernel's
  // critical path of dependent loads).
  double gphi_i = 0, gphi_j = 0;
  int ci = -1, cj = -1;
  if (n < P) {
    PairGradOut o;
    pair_grad_one<KIND>(g, q, geo_split(g, params, R), sched[1], n, o);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      pg[k * P + n] = o.gRi[k];
      pg[(9 + k) * P + n] = o.gRj[k];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) pg[(18 + k) * P + n] = o.gdc[k];
    pg[21 * P + n] = o.gphi_i;
    pg[22 * P + n] = o.gphi_j;
    pg[23 * P + n] = o.loss;
    if (!isfinite(o.loss)) raise_flag(flag, FM_ERR_NONFINITE_LOSS);
    gphi_i = o.gphi_i;
    gphi_j = o.gphi_j;
    if (g.refine_focal) {
      ci = g.pair_ci[n];
      cj = g.pair_cj[n];
    }
  }
  if (cams_by_block(g)) {
    // per-camera sums of this block's focal terms: warp butterflies, then the
    // two warps in order (fixed order -> reproducible)
    __shared__ double wsum[kPairBlock / 32][kBlockCams];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int c = 0; c < g.n_cameras; ++c) {
      double v = (ci == c ? gphi_i : 0.0) + (cj == c ? gphi_j : 0.0);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) wsum[w][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < g.n_cameras) {
      double v = 0;
#pragma unroll
      for (int k = 0; k < kPairBlock / 32; ++k) v += wsum[k][threadIdx.x];
      cpart[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = v;
    }
  }
}


template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

__device__ __forceinline__ void adam_elem(double& p, double& m, double& v, double g, double lr,
                                          double b1, double b2, double eps, double bc1, double bc2) {
  const double mk = __dadd_rn(__dmul_rn(b1, m), __dmul_rn(1.0 - b1, g));
  const double vk = __dadd_rn(__dmul_rn(b2, v), __dmul_rn(1.0 - b2, __dmul_rn(g, g)));
  m = mk;
  v = vk;
  p = __dsub_rn(p, __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, bc1)), __dadd_rn(sqrt(__ddiv_rn(vk, bc2)), eps)));
}

struct AdamArgs {
  double* m;
  double* v;
  double b1, b2, eps;
  const double* sched;  // lr, scale, bc1[kMaxSteps], bc2[kMaxSteps]
  int step;             // index into the bias-correction table
};

// One launch, two roles.  Blocks [0, img_blocks): warp per image --
// fixed-order gather of the image's incidences, 6D VJP (every lane computes it
// redundantly from the butterfly-reduced totals), then either the packed
// gradient (API) or Adam with lane q updating parameter q, and the new
// rotation.  Blocks [img_blocks, ..): one block per camera chunk --
// fixed-order partial sum of focal gradients (ref/epipolar.py:194-196).
constexpr int kReduceBlock = 64;  // 2 warps: spreads small image counts over all SMs

// Camera c's focal gradient `acc` (lane 0): the packed gradient (API) or
// Adam and the focal scale the next step's pairs read.
template <bool ADAM>
__device__ __forceinline__ void cam_update(const fm_pair_graph& g, double* __restrict__ params,
                                           double* F, double* __restrict__ grad, const AdamArgs& ad,
                                           int32_t* flag, int c, double acc) {
  const int idx = 9 * g.n_images + c;
  if (!ADAM) {
    grad[idx] = acc;
    return;
  }
  if (!isfinite(acc)) {
    raise_flag(flag, FM_ERR_NONFINITE_GRAD);
    return;
  }
  const double lr = ad.sched[0];
  const double bc1 = ad.sched[2 + ad.step], bc2 = ad.sched[2 + kMaxSteps + ad.step];
  adam_elem(params[idx], ad.m[idx], ad.v[idx], acc, lr, ad.b1, ad.b2, ad.eps, bc1, bc2);
  F[c] = exp(-params[idx]);  // the focal scale the next step's pairs read
}

template <bool ADAM>
__device__ void cam_finalise(const fm_pair_graph& g, double* __restrict__ params, double* R,
                             const double* __restrict__ cpart, double* __restrict__ grad,
                             const AdamArgs& ad, int32_t* flag) {
  // Executed by the last camera-chunk block: warp per camera, fixed-order
  // lane-strided sum of the chunk partials + butterfly, then Adam.
  const int lane = threadIdx.x & 31;
  for (int c = threadIdx.x >> 5; c < g.n_cameras; c += kReduceBlock / 32) {
    double acc = 0;
    for (int k = g.cam_chunk_off[c] + lane; k < g.cam_chunk_off[c + 1]; k += 32) acc += __ldcg(cpart + k);
    acc = warp_sum(acc);
    if (lane == 0) cam_update<ADAM>(g, params, R + 9 * (int64_t)g.n_images, grad, ad, flag, c, acc);
  }
}

// ---- image_reduce building blocks (shared with the peer-exchange kernel)

// Camera c's focal gradient from pair_grad's per-block partials cpart[c][..]:
// a fixed lane-strided order + butterfly (every lane returns the sum).  All
// of a lane's partials are in flight at once (up to 32 x 16 per batch).
__device__ __forceinline__ double cam_block_sum(const fm_pair_graph& g, const double* __restrict__ cpart,
                                                int c, int lane) {
  const int64_t P = g.n_pairs;
  const int64_t nb = (P + kPairBlock - 1) / kPairBlock;
  const double* part = cpart + (int64_t)c * nb;
  constexpr int kB = 16;
  double acc = 0;
  for (int64_t k0 = 0; k0 < nb; k0 += 32 * kB) {
    double v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t k = k0 + lane + 32 * u;
      v[u] = k < nb ? part[k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (k0 + lane + 32 * u < nb) acc += v[u];
  }
  return warp_sum(acc);
}

// Image k's packed-gradient component owned by this lane (lanes 0..5: the 6D
// rotation parameters, 6..8: the centre) and whether the image's gradient is
// finite (ref/optim.py:28-29).  Fixed-order gather of the image's incidences
// (batches of kGather per lane: all index loads, then all gradient loads in
// flight, then the adds in incidence order -- the order of a plain loop over
// e0 + lane, e0 + lane + 32, ...; the first batch from the padded table
// inc_pad, so it does not wait for img_off), butterfly sums, 6D VJP.
struct ImageGrad {
  double gq;
  bool ok;
};
__device__ __forceinline__ ImageGrad image_grad(const fm_pair_graph& g, const double* __restrict__ params,
                                                const double* __restrict__ pg,
                                                const int* __restrict__ inc_pad, int k, int lane) {
  const int64_t P = g.n_pairs;
  double acc[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = 0;
  constexpr int kGather = kIncPad / 32;
  auto gather = [&](const int (&inc)[kGather]) {
    double v[kGather][12];
#pragma unroll
    for (int u = 0; u < kGather; ++u) {
      const int64_t n = inc[u] >= 0 ? (inc[u] >> 1) : 0;
      const int base = (inc[u] & 1) ? 9 : 0;
#pragma unroll
      for (int q = 0; q < 9; ++q) v[u][q] = inc[u] >= 0 ? pg[(base + q) * P + n] : 0.0;
#pragma unroll
      for (int q = 0; q < 3; ++q) v[u][9 + q] = inc[u] >= 0 ? pg[(18 + q) * P + n] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kGather; ++u) {
      if (inc[u] < 0) break;
      const double sgn = (inc[u] & 1) ? 1.0 : -1.0;
#pragma unroll
      for (int q = 0; q < 9; ++q) acc[q] += v[u][q];
#pragma unroll
      for (int q = 0; q < 3; ++q) acc[9 + q] += sgn * v[u][9 + q];
    }
  };
  const int e0 = g.img_off[k], e1 = g.img_off[k + 1];  // needed only past the table
  {
    int inc[kGather];
#pragma unroll
    for (int u = 0; u < kGather; ++u) inc[u] = inc_pad[(int64_t)k * kIncPad + lane + 32 * u];
    gather(inc);
  }
  for (int eb = e0 + kIncPad + lane; eb < e1; eb += 32 * kGather) {
    int inc[kGather];
#pragma unroll
    for (int u = 0; u < kGather; ++u) inc[u] = eb + 32 * u < e1 ? g.img_inc[eb + 32 * u] : -1;
    gather(inc);
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) acc[q] = warp_sum(acc[q]);
  double vcur[6], g6[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) vcur[q] = params[6 * (int64_t)k + q];
  rot6d_vjp(vcur, acc, g6);
  ImageGrad r;
  r.gq = acc[9];
#pragma unroll
  for (int q = 0; q < 6; ++q) r.gq = lane == q ? g6[q] : r.gq;
  r.gq = lane == 7 ? acc[10] : (lane == 8 ? acc[11] : r.gq);
  r.ok = true;
#pragma unroll
  for (int q = 0; q < 6; ++q) r.ok = r.ok && isfinite(g6[q]);
#pragma unroll
  for (int q = 0; q < 3; ++q) r.ok = r.ok && isfinite(acc[9 + q]);
  return r;
}

// Adam on image k's nine parameters (lane q: parameter q, the numpy
// expression order) and its new rotation (lanes 0..5 feed rot6d_to_R).
// Whole warp.
__device__ __forceinline__ void image_adam(const fm_pair_graph& g, double* __restrict__ params,
                                           double* __restrict__ R, const AdamArgs& ad, int32_t* flag,
                                           int k, int lane, double gq) {
  const int N = g.n_images;
  const double lr = ad.sched[0];
  const double bc1 = ad.sched[2 + ad.step], bc2 = ad.sched[2 + kMaxSteps + ad.step];
  double newp = 0.0;
  if (lane < 9) {
    const int64_t idx = lane < 6 ? 6 * (int64_t)k + lane : 6 * (int64_t)N + 3 * k + (lane - 6);
    double pv = params[idx];
    adam_elem(pv, ad.m[idx], ad.v[idx], gq, lr, ad.b1, ad.b2, ad.eps, bc1, bc2);
    params[idx] = pv;
    newp = pv;
  }
  // new rotation from the six updated 6D parameters (lanes 0..5)
  double v6n[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) v6n[q] = __shfl_sync(0xffffffffu, newp, q);
  double Rk[9];
  const int code = rot6d_to_R(v6n, Rk);
  if (lane == 0 && code) raise_flag(flag, code);
  double val = Rk[0];
#pragma unroll
  for (int q = 1; q < 9; ++q) val = lane == q ? Rk[q] : val;
  if (lane < 9) R[9 * (int64_t)k + lane] = val;
}

// One launch, two roles.  Blocks [0, img_blocks): warp per image --
// image_grad (fixed-order gather, butterflies, 6D VJP), then either the
// packed gradient (API) or Adam with lane q updating parameter q and the new
// rotation (image_adam).  Blocks [img_blocks, ..): the focal gradients --
// with few cameras a warp per camera over pair_grad's block partials
// (cam_block_sum); otherwise a block per camera chunk, fixed-order partial
// sums, and the last chunk block to finish (atomic ticket) sums the partials
// per camera in chunk order and applies the focal update
// (ref/epipolar.py:194-196).
template <bool ADAM>
__global__ void __launch_bounds__(kReduceBlock, 8)  // <= 128 registers: 8 blocks/SM (C4: one wave)
image_reduce_kernel(const fm_pair_graph g, double* __restrict__ params,
                    const double* __restrict__ pg, double* __restrict__ grad,
                    double* __restrict__ R, double* __restrict__ cpart, unsigned int* ticket,
                    const int img_blocks, const AdamArgs ad, int32_t* flag,
                    const int* __restrict__ inc_pad, double* __restrict__ nonfinite_out) {
  __shared__ double red[kReduceBlock];
  __shared__ bool last;
  const int64_t P = g.n_pairs;
  if ((int)blockIdx.x >= img_blocks && cams_by_block(g)) {  // ---- camera role, few cameras
    const int c = ((int)blockIdx.x - img_blocks) * (kReduceBlock / 32) + (threadIdx.x >> 5);
    if (c >= g.n_cameras) return;
    const int lane = threadIdx.x & 31;
    const double acc = cam_block_sum(g, cpart, c, lane);
    if (ADAM && *flag) return;  // checked after the loads: off their critical path
    if (lane == 0) cam_update<ADAM>(g, params, R + 9 * (int64_t)g.n_images, grad, ad, flag, c, acc);
    return;
  }
  if ((int)blockIdx.x >= img_blocks) {  // ---- camera chunk role
    const int c = blockIdx.x - img_blocks;
    // a raised flag skips the work but never the ticket: every chunk block
    // counts, so the last one always re-arms it (the flag can be raised by
    // image blocks of this same launch)
    const bool skip = ADAM && *flag;
    double acc = 0;
    const int lo = g.cam_chunk_lo[c], hi = skip ? lo : g.cam_chunk_lo[c + 1];
    // unrolled: the two dependent loads of several incidences in flight
    // together (same per-thread accumulation order)
#pragma unroll 8
    for (int e = lo + threadIdx.x; e < hi; e += kReduceBlock) {
      const int inc = g.cam_inc[e];
      acc += pg[(21 + (inc & 1)) * P + (inc >> 1)];
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = kReduceBlock / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      cpart[c] = red[0];
      __threadfence();
      last = atomicAdd(ticket, 1u) == (unsigned)(gridDim.x - img_blocks - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (!(ADAM && *(volatile int32_t*)flag)) cam_finalise<ADAM>(g, params, R, cpart, grad, ad, flag);
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next step
    return;
  }
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int N = g.n_images;
  if (k >= N) return;
  const ImageGrad ig = image_grad(g, params, pg, inc_pad, k, lane);
  if (!ADAM) {
    if (lane < 6) grad[6 * (int64_t)k + lane] = ig.gq;
    else if (lane < 9) grad[6 * (int64_t)N + 3 * k + lane - 6] = ig.gq;
    // sharded step: this rank's pair_grad saw a non-finite loss term -> a NaN
    // in the all-reduced buffer makes every rank raise the loss error
    if (nonfinite_out && k == 0 && lane == 0)
      *nonfinite_out = *flag == FM_ERR_NONFINITE_LOSS ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
    return;
  }
  if (*flag) return;  // a raised flag freezes the parameters (checked late: off the load chain)
  if (!ig.ok) {
    if (lane == 0) raise_flag(flag, FM_ERR_NONFINITE_GRAD);
    return;
  }
  image_adam(g, params, R, ad, flag, k, lane, ig.gq);
}

// ------------------------------------------------ fused gradient exchange
// The sharded step's reduce fused with its collective, over peer
// memory instead of a separate all-reduce: every rank runs this kernel on
// its own pair shard at the same time.  A logical block (2 images, or 2
// cameras) computes its local packed-gradient components (image_grad /
// cam_block_sum, exactly the sharded API path's values), writes them to its
// rank's exchange buffer, publishes the step id on its own ready flag
// (st.release.sys), waits until every peer has published the same logical
// block (ld.acquire.sys), sums the ranks' components in rank order -- the
// same sum on every rank, so the replicated parameters stay bitwise equal
// -- and applies Adam.  No grid barrier and no second kernel: blocks
// synchronise pairwise with their peers.  One physical block per resident
// slot walks the logical blocks in order (every rank the same order), so
// the waits cannot deadlock.  Buffers are double-buffered by step parity: a
// rank can only reach step s+1 after every peer published step s, i.e.
// finished reading step s-1's buffer.  A non-finite loss term on any rank
// travels as a NaN marker per logical block; spins are bounded (a peer that
// never arrives raises FM_ERR_CUDA instead of hanging the GPU).
// SYS: peers on other GPUs (system scope); else ranks sharing this GPU.
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
template <bool SYS>
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  if (SYS) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
  else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct PeerArgs {
  int n_ranks, rank;
  double* const* part;             // [n_ranks] exchange buffers [2][n_pub]
  unsigned long long* const* ready;  // [n_ranks] flag arrays [n_logical]
  int64_t n_pub;                   // 9N + C + n_logical (components + NaN markers)
  int sys;                         // peers on other GPUs: system-scope ordering
};

template <bool SYS>
__global__ void __launch_bounds__(kReduceBlock, 8)
image_reduce_peer_kernel(const fm_pair_graph g, double* __restrict__ params,
                         const double* __restrict__ pg, double* __restrict__ R,
                         const double* __restrict__ cpart, const int img_blocks, const int n_logical,
                         const AdamArgs ad, int32_t* flag, const int* __restrict__ inc_pad,
                         const PeerArgs pa) {
  __shared__ int marker_bad;
  const int N = g.n_images;
  const int n_cam = g.refine_focal ? g.n_cameras : 0;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned long long step_id = (unsigned long long)ad.sched[2 + 2 * kMaxSteps] + ad.step + 1;
  const int parity = (int)(step_id & 1);
  const int local_bad = *flag == FM_ERR_NONFINITE_LOSS;  // this rank's pair terms (pair_grad done)
  double* mine = pa.part[pa.rank] + parity * pa.n_pub;
  const int64_t marker0 = (int64_t)9 * N + n_cam;
  for (int b = blockIdx.x; b < n_logical; b += gridDim.x) {
    // ---- local components and their slots
    int64_t slot = -1;  // this lane's published slot (-1: none)
    double val = 0.0;
    if (b < img_blocks) {
      const int k = b * (kReduceBlock / 32) + w;
      if (k < N) {
        const ImageGrad ig = image_grad(g, params, pg, inc_pad, k, lane);
        if (lane < 6) slot = 6 * (int64_t)k + lane;
        else if (lane < 9) slot = 6 * (int64_t)N + 3 * k + lane - 6;
        val = ig.gq;
      }
    } else {
      const int c = (b - img_blocks) * (kReduceBlock / 32) + w;
      if (c < n_cam) {
        const double acc = cam_block_sum(g, cpart, c, lane);
        if (lane == 0) {
          slot = 9 * (int64_t)N + c;
          val = acc;
        }
      }
    }
    if (slot >= 0) mine[slot] = val;
    if (threadIdx.x == 0) mine[marker0 + b] = local_bad ? __longlong_as_double(0x7ff8000000000000ll) : 0.0;
    __syncthreads();
    // ---- publish, then wait for every peer's same logical block
    // the release store orders the whole block's writes (cumulative through
    // the barrier above): no separate system-scope fence
    if (threadIdx.x == 0) st_release<SYS>(pa.ready[pa.rank] + b, step_id);
    if ((int)threadIdx.x < pa.n_ranks) {
      const unsigned long long* f = pa.ready[threadIdx.x] + b;
      long long spins = 0;
      while (ld_acquire<SYS>(f) < step_id) {
        __nanosleep(64);
        // a peer that never arrives (~1 s) raises FM_ERR_CUDA once; after
        // that nobody waits any more, so the launch drains instead of hanging
        if ((++spins & 1023) == 0 &&
            (*(volatile int32_t*)flag == FM_ERR_CUDA || spins > (1ll << 24))) {
          atomicCAS(flag, 0, FM_ERR_CUDA);
          break;
        }
      }
    }
    __syncthreads();
    // ---- rank-order sums (identical on every rank)
    double tot = 0.0, bad = 0.0;
    for (int r = 0; r < pa.n_ranks; ++r) {
      const double* pr = pa.part[r] + parity * pa.n_pub;
      if (slot >= 0) tot += __ldcv(pr + slot);
      bad += __ldcv(pr + marker0 + b);
    }
    if (threadIdx.x == 0) marker_bad = !(bad == bad) ? 1 : 0;  // NaN marker from some rank
    __syncthreads();
    const bool loss_bad = marker_bad != 0;
    __syncthreads();  // marker_bad is rewritten by the next logical block
    if (loss_bad) {
      if (threadIdx.x == 0) raise_flag(flag, FM_ERR_NONFINITE_LOSS);
      continue;
    }
    if (*(volatile int32_t*)flag) continue;  // frozen (every rank alike)
    if (b < img_blocks) {
      const int k = b * (kReduceBlock / 32) + w;
      if (k >= N) continue;
      // the summed gradient's finiteness decides (ref/optim.py:28-29), as
      // after the all-reduce of the other sharded paths
      bool fin = (lane >= 9) || isfinite(tot);
      fin = __all_sync(0xffffffffu, fin);
      if (!fin) {
        if (lane == 0) raise_flag(flag, FM_ERR_NONFINITE_GRAD);
        continue;
      }
      image_adam(g, params, R, ad, flag, k, lane, tot);
    } else {
      const int c = (b - img_blocks) * (kReduceBlock / 32) + w;
      if (c < n_cam && lane == 0) cam_update<true>(g, params, R + 9 * (int64_t)N, nullptr, ad, flag, c, tot);
    }
  }
}

// Replicated Adam of the sharded engine (ref/optim.py:24-36) over the
// all-reduced packed gradient + loss `gbuf` [9N + C | loss]: blocks
// [0, img_blocks) warp per image -- lanes 0..8 update the image's nine
// parameters with the single-GPU expression (adam_elem), lanes 0..5 feed the
// new rotation the next step's pairs read; the remaining blocks a thread per
// camera (focal parameter + its scale exp(-log_focal)).  Checks follow
// ref/epipolar.py:306-307 (loss) then ref/optim.py:28-29 (gradient).
__global__ void __launch_bounds__(kReduceBlock)
adam_dist_kernel(const fm_pair_graph g, double* __restrict__ params, const double* __restrict__ gbuf,
                 double* __restrict__ R, const AdamArgs ad, int32_t* flag, const int img_blocks) {
  if (*flag) return;
  const int N = g.n_images;
  const int n_cam = g.refine_focal ? g.n_cameras : 0;
  const double loss = gbuf[(int64_t)9 * N + n_cam];
  if (!isfinite(loss)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_flag(flag, FM_ERR_NONFINITE_LOSS);
    return;
  }
  const double lr = ad.sched[0];
  const double bc1 = ad.sched[2 + ad.step], bc2 = ad.sched[2 + kMaxSteps + ad.step];
  if ((int)blockIdx.x >= img_blocks) {
    const int c = ((int)blockIdx.x - img_blocks) * blockDim.x + threadIdx.x;
    if (c >= n_cam) return;
    const int64_t idx = (int64_t)9 * N + c;
    const double gq = gbuf[idx];
    if (!isfinite(gq)) {
      raise_flag(flag, FM_ERR_NONFINITE_GRAD);
      return;
    }
    adam_elem(params[idx], ad.m[idx], ad.v[idx], gq, lr, ad.b1, ad.b2, ad.eps, bc1, bc2);
    R[idx] = exp(-params[idx]);
    return;
  }
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= N) return;
  const int64_t idx = lane < 6 ? 6 * (int64_t)k + lane : 6 * (int64_t)N + 3 * k + (lane - 6);
  const double gq = lane < 9 ? gbuf[idx] : 0.0;
  if (!__all_sync(0xffffffffu, lane >= 9 || isfinite(gq))) {
    if (lane == 0) raise_flag(flag, FM_ERR_NONFINITE_GRAD);
    return;
  }
  double newp = 0.0;
  if (lane < 9) {
    double pv = params[idx];
    adam_elem(pv, ad.m[idx], ad.v[idx], gq, lr, ad.b1, ad.b2, ad.eps, bc1, bc2);
    params[idx] = pv;
    newp = pv;
  }
  double v6n[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) v6n[q] = __shfl_sync(0xffffffffu, newp, q);
  double Rk[9];
  const int code = rot6d_to_R(v6n, Rk);
  if (lane == 0 && code) raise_flag(flag, code);
  double val = Rk[0];
#pragma unroll
  for (int q = 1; q < 9; ++q) val = lane == q ? Rk[q] : val;
  if (lane < 9) R[9 * (int64_t)k + lane] = val;
}

// inc_pad[k][t] = image k's incidence t (t < degree), else -1: image_reduce's
// first gather batch reads it without waiting for img_off.
__global__ void inc_pad_kernel(const fm_pair_graph g, int* __restrict__ inc_pad) {
  const int k = blockIdx.x;
  const int e0 = g.img_off[k], deg = g.img_off[k + 1] - e0;
  for (int t = threadIdx.x; t < kIncPad; t += blockDim.x)
    inc_pad[(int64_t)k * kIncPad + t] = t < deg ? g.img_inc[e0 + t] : -1;
}

int build_inc_pad(const fm_pair_graph& g, const EpiScratch& s, cudaStream_t st) {
  if (g.n_images == 0) return FM_OK;
  inc_pad_kernel<<<(unsigned)g.n_images, kIncPad, 0, st>>>(g, s.inc_pad);
  FM_LAUNCHED(inc_pad_kernel);
  return FM_OK;
}

// Deterministic two-level sum of the per-pair loss terms.
__global__ void loss_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[256];
  double acc = 0;
  for (int64_t k = blockIdx.x * 256 + threadIdx.x; k < n; k += (int64_t)gridDim.x * 256) acc += x[k];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void loss_final_kernel(const double* __restrict__ part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double acc = 0;
    for (int k = 0; k < nb; ++k) acc += part[k];
    *out = acc;
  }
}

// scale = 2/Z from a pass's fused totals {L1, Z, kept} (device), so the host
// need not read Z back between the pass and the epoch (ref/epipolar.py:291,
// `2.0 / Z` with Z an integer count: the same IEEE division)
__global__ void sched_scale_kernel(double* sched, const double* totals) { sched[1] = 2.0 / totals[1]; }

// Pinned staging for the per-call schedule upload: a pageable
// cudaMemcpyAsync may wait for the stream, which would serialise the host
// with the device between epochs.  A small ring of pinned buffers, each
// reused only after its previous copy completed (event).
constexpr int kSchedLen = 3 + 2 * kMaxSteps;
struct PinnedSched {
  double* host = nullptr;
  cudaEvent_t done = nullptr;
};
std::mutex g_pin_mu;
PinnedSched g_pin[8];
int g_pin_next = 0;

int upload_sched(const std::vector<double>& sched, double* dst, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_pin_mu);
  PinnedSched& slot = g_pin[g_pin_next];
  g_pin_next = (g_pin_next + 1) % 8;
  if (!slot.host) {
    FM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&slot.host), kSchedLen * sizeof(double)));
    FM_CUDA(cudaEventCreateWithFlags(&slot.done, cudaEventDisableTiming));
  } else {
    FM_CUDA(cudaEventSynchronize(slot.done));  // its previous copy has been consumed
  }
  memcpy(slot.host, sched.data(), kSchedLen * sizeof(double));
  FM_CUDA(cudaMemcpyAsync(dst, slot.host, kSchedLen * sizeof(double), cudaMemcpyHostToDevice, st));
  FM_CUDA(cudaEventRecord(slot.done, st));
  return FM_OK;
}

__global__ void set_sched_kernel(double* sched, double lr, double scale, unsigned int* ticket) {
  sched[0] = lr;
  sched[1] = scale;
  *ticket = 0u;
}

int launch_pair_grad(const fm_pair_graph& g, const fm_quad_model& q, const double* params,
                     const EpiScratch& s, int32_t* flag, cudaStream_t st) {
  const unsigned blocks = (unsigned)pair_blocks(g);
  switch (q.kind) {
    case FM_QUAD_SHIFTED32:
      pair_grad_kernel<FM_QUAD_SHIFTED32><<<blocks, kPairBlock, 0, st>>>(g, q, params, s.R, s.sched, s.pg, s.cpart,
                                                                    flag);
      break;
    case FM_QUAD_W64:
      pair_grad_kernel<FM_QUAD_W64><<<blocks, kPairBlock, 0, st>>>(g, q, params, s.R, s.sched, s.pg, s.cpart,
                                                                    flag);
      break;
    case FM_QUAD_MOM64:
      pair_grad_kernel<FM_QUAD_MOM64><<<blocks, kPairBlock, 0, st>>>(g, q, params, s.R, s.sched, s.pg, s.cpart,
                                                                    flag);
      break;
    default:
      return set_error(FM_ERR_INVALID, "unknown quadratic model kind %d", q.kind);
  }
  FM_LAUNCHED(pair_grad_kernel);
  return FM_OK;
}

int check_graph(const fm_pair_graph* g) {
  FM_REQUIRE(g, "null pair graph");
  FM_REQUIRE(g->n_images >= 0 && g->n_pairs >= 0 && g->n_cameras >= 0, "negative graph sizes");
  FM_REQUIRE(!g->refine_focal || g->n_cameras > 0, "refine_focal needs n_cameras > 0");
  return FM_OK;
}

int check_quad(const fm_quad_model* q) {
  FM_REQUIRE(q, "null quadratic model");
  if (q->kind == FM_QUAD_SHIFTED32)
    FM_REQUIRE(q->mom32 && q->vgrad && q->s0 && q->ghat0, "incomplete shifted model");
  else if (q->kind == FM_QUAD_W64)
    FM_REQUIRE(q->w81, "missing dense W");
  else if (q->kind == FM_QUAD_MOM64)
    FM_REQUIRE(q->mom64, "missing fp64 moments");
  else
    return set_error(FM_ERR_INVALID, "unknown quadratic model kind %d", q->kind);
  return FM_OK;
}

// Enqueue n_steps optimizer steps (kernels only, no host work) on `st`.
int enqueue_steps(const fm_pair_graph& g, const fm_quad_model& q, double* params, double* m,
                  double* v, int n_steps, double b1, double b2, double eps, const EpiScratch& s,
                  int32_t* flag, cudaStream_t st) {
  const int N = g.n_images;
  for (int step = 0; step < n_steps; ++step) {
    int rc = launch_pair_grad(g, q, params, s, flag, st);
    if (rc) return rc;
    AdamArgs ad{m, v, b1, b2, eps, s.sched, step};
    const int img_blocks = (int)ceil_div((int64_t)N * 32, kReduceBlock);
    const int cam_blocks = cam_role_blocks(g);
    if (img_blocks + cam_blocks > 0) {
      image_reduce_kernel<true><<<(unsigned)(img_blocks + cam_blocks), kReduceBlock, 0, st>>>(
          g, params, s.pg, nullptr, s.R, s.cpart, s.ticket, img_blocks, ad, flag, s.inc_pad, nullptr);
      FM_LAUNCHED(image_reduce_kernel);
    }
  }
  return FM_OK;
}

// Sharded form of enqueue_steps: per step the local pairs' packed gradient
// and loss (the API kernels, fm_epi_loss_grad's), one all-reduce of
// [9N + C | loss] over `comm`, then the replicated Adam step.
int enqueue_steps_dist(const fm_pair_graph& g, const fm_quad_model& q, double* params, double* m,
                       double* v, int n_steps, double b1, double b2, double eps, const EpiScratch& s,
                       int32_t* flag, void* comm, double* gbuf, cudaStream_t st) {
  const int N = g.n_images;
  const int64_t P = g.n_pairs;
  const int n_cam = g.refine_focal ? g.n_cameras : 0;
  const size_t n_grad = (size_t)9 * N + n_cam;
  const int img_blocks = (int)ceil_div((int64_t)N * 32, kReduceBlock);
  const int cam_blocks = cam_role_blocks(g);
  for (int step = 0; step < n_steps; ++step) {
    AdamArgs none{nullptr, nullptr, 0, 0, 0, s.sched, step};
    if (P > 0) {
      if (int rc = launch_pair_grad(g, q, params, s, flag, st)) return rc;
      // the loss slot gbuf[n_grad] carries only its finiteness (0 or NaN,
      // written by image_reduce): the step needs no loss value
      if (img_blocks + cam_blocks > 0) {
        image_reduce_kernel<false><<<(unsigned)(img_blocks + cam_blocks), kReduceBlock, 0, st>>>(
            g, params, s.pg, gbuf, s.R, s.cpart, s.ticket, img_blocks, none, flag, s.inc_pad,
            gbuf + n_grad);
        FM_LAUNCHED(image_reduce_kernel);
      }
    } else {  // a rank without pairs contributes zeros
      FM_CUDA(cudaMemsetAsync(gbuf, 0, (n_grad + 1) * sizeof(double), st));
    }
    if (int rc = nccl_allreduce_sum_f64(gbuf, n_grad + 1, comm, st)) return rc;
    AdamArgs ad{m, v, b1, b2, eps, s.sched, step};
    const int cb = (int)ceil_div(n_cam, kReduceBlock);
    if (img_blocks + cb > 0) {
      adam_dist_kernel<<<(unsigned)(img_blocks + cb), kReduceBlock, 0, st>>>(g, params, gbuf, s.R, ad, flag,
                                                                            img_blocks);
      FM_LAUNCHED(adam_dist_kernel);
    }
  }
  return FM_OK;
}

// The peer-exchange step: pair_grad, then the fused reduce + exchange + Adam.
int enqueue_steps_peer(const fm_pair_graph& g, const fm_quad_model& q, double* params, double* m,
                       double* v, int n_steps, double b1, double b2, double eps, const EpiScratch& s,
                       int32_t* flag, const PeerArgs& pa, int grid, cudaStream_t st) {
  const int N = g.n_images;
  const int img_blocks = (int)ceil_div((int64_t)N * 32, kReduceBlock);
  const int n_logical = img_blocks + (cams_by_block(g) ? (int)ceil_div(g.n_cameras, 2) : 0);
  for (int step = 0; step < n_steps; ++step) {
    if (g.n_pairs > 0)
      if (int rc = launch_pair_grad(g, q, params, s, flag, st)) return rc;
    AdamArgs ad{m, v, b1, b2, eps, s.sched, step};
    if (pa.sys)
      image_reduce_peer_kernel<true><<<(unsigned)grid, kReduceBlock, 0, st>>>(
          g, params, s.pg, s.R, s.cpart, img_blocks, n_logical, ad, flag, s.inc_pad, pa);
    else
      image_reduce_peer_kernel<false><<<(unsigned)grid, kReduceBlock, 0, st>>>(
          g, params, s.pg, s.R, s.cpart, img_blocks, n_logical, ad, flag, s.inc_pad, pa);
    FM_LAUNCHED(image_reduce_peer_kernel);
  }
  return FM_OK;
}

// --------------------------------------------------------------- graph cache
struct GraphKey {
  std::vector<uintptr_t> k;
  bool operator<(const GraphKey& o) const { return k < o.k; }
};
std::mutex g_graph_mu;
std::map<GraphKey, cudaGraphExec_t> g_graphs;

GraphKey make_key(const fm_pair_graph& g, const fm_quad_model& q, double* params, double* m,
                  double* v, int n_steps, double b1, double b2, double eps, const EpiScratch& s,
                  int32_t* flag) {
  GraphKey key;
  auto put = [&](const void* p) { key.k.push_back(reinterpret_cast<uintptr_t>(p)); };
  auto putd = [&](double d) {
    uintptr_t u = 0;
    memcpy(&u, &d, sizeof(d));
    key.k.push_back(u);
  };
  key.k.push_back((uintptr_t)g.n_images);
  key.k.push_back((uintptr_t)g.n_cameras);
  key.k.push_back((uintptr_t)g.refine_focal);
  key.k.push_back((uintptr_t)g.n_cam_chunks);
  key.k.push_back((uintptr_t)g.n_pairs);
  for (const void* p : {(const void*)g.pair_i, (const void*)g.pair_j, (const void*)g.pair_ci,
                        (const void*)g.pair_cj, (const void*)g.img_off, (const void*)g.img_inc,
                        (const void*)g.cam_off, (const void*)g.cam_inc, (const void*)g.cam_chunk_lo,
                        (const void*)g.cam_chunk_cam, (const void*)g.cam_chunk_off})
    put(p);
  key.k.push_back((uintptr_t)q.kind);
  for (const void* p : {(const void*)q.mom32, (const void*)q.vgrad, (const void*)q.s0,
                        (const void*)q.ghat0, (const void*)q.w81, (const void*)q.mom64})
    put(p);
  put(params);
  put(m);
  put(v);
  key.k.push_back((uintptr_t)n_steps);
  putd(b1);
  putd(b2);
  putd(eps);
  put(s.R);
  put(s.sched);
  put(flag);
  return key;
}

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_epi_scratch_bytes(const fm_pair_graph* g) { return g ? scratch_need(*g) : 0; }

int fm_epi_pair_ghat(const fm_pair_graph* g, const double* params, double* ghat, int32_t* flag,
                     void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = check_graph(g)) return rc;
  EpiScratch s;
  FM_REQUIRE(carve(*g, scratch, scratch_bytes, s), "epipolar scratch too small");
  cudaStream_t st = as_stream(stream);
  if (int rc = launch_image_rot(*g, params, s.R, flag, st)) return rc;
  if (g->n_pairs > 0) {
    pair_ghat_kernel<<<(unsigned)ceil_div(g->n_pairs, 128), 128, 0, st>>>(*g, params, s.R, ghat);
    FM_LAUNCHED(pair_ghat_kernel);
  }
  return FM_OK;
}

int fm_epi_loss_grad(const fm_pair_graph* g, const fm_quad_model* q, const double* params,
                     double scale, double* loss_out, double* grad_out, int32_t* flag, void* scratch,
                     size_t scratch_bytes, void* stream) {
  if (int rc = check_graph(g)) return rc;
  if (int rc = check_quad(q)) return rc;
  EpiScratch s;
  FM_REQUIRE(carve(*g, scratch, scratch_bytes, s), "epipolar scratch too small");
  cudaStream_t st = as_stream(stream);
  const int N = g->n_images;
  const int64_t P = g->n_pairs;
  const size_t n_grad = (size_t)9 * N + (g->refine_focal ? g->n_cameras : 0);
  set_sched_kernel<<<1, 1, 0, st>>>(s.sched, 0.0, scale, s.ticket);
  FM_LAUNCHED(set_sched_kernel);
  if (int rc = launch_image_rot(*g, params, s.R, flag, st)) return rc;
  if (P == 0) {
    FM_CUDA(cudaMemsetAsync(grad_out, 0, n_grad * sizeof(double), st));
    FM_CUDA(cudaMemsetAsync(loss_out, 0, sizeof(double), st));
    return FM_OK;
  }
  // API semantics: evaluate even if `flag` is already set by the caller
  if (int rc = build_inc_pad(*g, s, st)) return rc;
  if (int rc = launch_pair_grad(*g, *q, params, s, nullptr, st)) return rc;
  AdamArgs none{nullptr, nullptr, 0, 0, 0, s.sched, 0};
  {
    const int img_blocks = (int)ceil_div((int64_t)N * 32, kReduceBlock);
    const int cam_blocks = cam_role_blocks(*g);
    if (img_blocks + cam_blocks > 0) {
      image_reduce_kernel<false><<<(unsigned)(img_blocks + cam_blocks), kReduceBlock, 0, st>>>(
          *g, const_cast<double*>(params), s.pg, grad_out, s.R, s.cpart, s.ticket, img_blocks,
          none, flag, s.inc_pad, nullptr);
      FM_LAUNCHED(image_reduce_kernel);
    }
  }
  const int nb = loss_blocks(P);
  loss_partial_kernel<<<nb, 256, 0, st>>>(s.pg + (size_t)23 * P, P, s.lpart);
  FM_LAUNCHED(loss_partial_kernel);
  loss_final_kernel<<<1, 32, 0, st>>>(s.lpart, nb, loss_out);
  FM_LAUNCHED(loss_final_kernel);
  return FM_OK;
}

}  // extern "C"

extern "C" size_t fm_peer_part_len(const fm_pair_graph* g);

namespace fm {
namespace {
// Physical blocks of the peer kernel: every logical block, capped by what
// is resident at once (the waits need every block of every rank resident)
// and by the caller's max_blocks (ranks sharing one GPU in tests).
int peer_grid(const fm_pair_graph& g, const fm_peer_group* peer) {
  const int img_blocks = (int)ceil_div((int64_t)g.n_images * 32, kReduceBlock);
  const int n_logical = img_blocks + (cams_by_block(g) ? (int)ceil_div(g.n_cameras, 2) : 0);
  static int per_sm = 0;
  if (!per_sm) {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, image_reduce_peer_kernel<true>, kReduceBlock, 0);
    per_sm = b > 0 ? b : 1;
  }
  int grid = std::min(n_logical, per_sm * sm_count());
  if (peer->max_blocks > 0) grid = std::min(grid, (int)peer->max_blocks);
  return std::max(grid, 1);
}

// dist: the sharded step (comm may be NULL = one rank; gbuf [9N + C + 1]).
int adam_steps_impl(const fm_pair_graph* g, const fm_quad_model* q, double* params, double* adam_m,
                    double* adam_v, int64_t t0, int32_t n_steps, double lr, double beta1,
                    double beta2, double eps, double scale, int32_t* flag, int32_t use_graph,
                    void* scratch, size_t scratch_bytes, void* stream, bool dist, void* comm,
                    double* gbuf, const fm_peer_group* peer = nullptr,
                    const double* totals = nullptr) {
  if (int rc = check_graph(g)) return rc;
  if (int rc = check_quad(q)) return rc;
  FM_REQUIRE(flag, "fm_epi_adam_steps needs a device flag word");
  FM_REQUIRE(n_steps >= 0 && t0 >= 0, "bad step range");
  EpiScratch s;
  FM_REQUIRE(carve(*g, scratch, scratch_bytes, s), "epipolar scratch too small");
  cudaStream_t st = as_stream(stream);
  if (n_steps == 0) return FM_OK;
  FM_CUDA(cudaMemsetAsync(s.ticket, 0, sizeof(unsigned int), st));
  if (int rc = build_inc_pad(*g, s, st)) return rc;
  if (int rc = launch_image_rot(*g, params, s.R, flag, st)) return rc;
  for (int32_t done = 0; done < n_steps;) {
    const int chunk = std::min<int32_t>(n_steps - done, kMaxSteps);
    // schedule: lr, 2/Z, and the bias corrections 1 - beta^t computed with the
    // host pow() exactly as ref/optim.py:34-35 does
    std::vector<double> sched(kSchedLen, 1.0);
    sched[0] = lr;
    sched[1] = scale;
    sched[2 + 2 * kMaxSteps] = peer ? (double)(peer->epoch + done) : 0.0;  // peer step ids
    for (int k = 0; k < chunk; ++k) {
      const double t = (double)(t0 + done + k + 1);
      sched[2 + k] = 1.0 - pow(beta1, t);
      sched[2 + kMaxSteps + k] = 1.0 - pow(beta2, t);
    }
    if (int rc = upload_sched(sched, s.sched, st)) return rc;
    if (totals) {
      sched_scale_kernel<<<1, 1, 0, st>>>(s.sched, totals);
      FM_LAUNCHED(sched_scale_kernel);
    }
    auto enqueue = [&](cudaStream_t cs) {
      if (peer) {
        PeerArgs pa{peer->n_ranks, peer->rank, peer->part, peer->ready,
                    (int64_t)fm_peer_part_len(g), peer->system_scope != 0};
        return enqueue_steps_peer(*g, *q, params, adam_m, adam_v, chunk, beta1, beta2, eps, s, flag,
                                  pa, peer_grid(*g, peer), cs);
      }
      return dist ? enqueue_steps_dist(*g, *q, params, adam_m, adam_v, chunk, beta1, beta2, eps, s,
                                       flag, comm, gbuf, cs)
                  : enqueue_steps(*g, *q, params, adam_m, adam_v, chunk, beta1, beta2, eps, s, flag, cs);
    };
    if (!use_graph) {
      if (int rc = enqueue(st)) return rc;
    } else {
      GraphKey key = make_key(*g, *q, params, adam_m, adam_v, chunk, beta1, beta2, eps, s, flag);
      key.k.push_back(dist ? 1u : (peer ? 2u : 0u));
      if (peer) {
        key.k.push_back(reinterpret_cast<uintptr_t>(peer->part));
        key.k.push_back(reinterpret_cast<uintptr_t>(peer->ready));
        key.k.push_back((uintptr_t)peer->n_ranks);
        key.k.push_back((uintptr_t)peer->rank);
        key.k.push_back((uintptr_t)peer->max_blocks);
        key.k.push_back((uintptr_t)peer->system_scope);
      }
      key.k.push_back(reinterpret_cast<uintptr_t>(comm));
      key.k.push_back(reinterpret_cast<uintptr_t>(gbuf));
      cudaGraphExec_t exec = nullptr;
      {
        std::lock_guard<std::mutex> lk(g_graph_mu);
        auto it = g_graphs.find(key);
        if (it != g_graphs.end()) exec = it->second;
      }
      if (!exec) {
        cudaStream_t cs;
        FM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FM_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue(cs);
        cudaGraph_t graph = nullptr;
        cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        if (rc) {
          if (graph) cudaGraphDestroy(graph);
          return rc;
        }
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture", __FILE__, __LINE__);
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate", __FILE__, __LINE__);
        std::lock_guard<std::mutex> lk(g_graph_mu);
        if (g_graphs.size() >= 16) {
          for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second);
          g_graphs.clear();
        }
        g_graphs[key] = exec;
      }
      FM_CUDA(cudaGraphLaunch(exec, st));
    }
    done += chunk;
  }
  return FM_OK;
}
}  // namespace
}  // namespace fm

extern "C" {

int fm_epi_adam_steps(const fm_pair_graph* g, const fm_quad_model* q, double* params,
                      double* adam_m, double* adam_v, int64_t t0, int32_t n_steps, double lr,
                      double beta1, double beta2, double eps, double scale, int32_t* flag,
                      int32_t use_graph, void* scratch, size_t scratch_bytes, void* stream) {
  return adam_steps_impl(g, q, params, adam_m, adam_v, t0, n_steps, lr, beta1, beta2, eps, scale,
                         flag, use_graph, scratch, scratch_bytes, stream, false, nullptr, nullptr);
}

int fm_epi_adam_steps_z(const fm_pair_graph* g, const fm_quad_model* q, double* params,
                        double* adam_m, double* adam_v, int64_t t0, int32_t n_steps, double lr,
                        double beta1, double beta2, double eps, const double* totals, int32_t* flag,
                        int32_t use_graph, void* scratch, size_t scratch_bytes, void* stream) {
  FM_REQUIRE(totals, "fm_epi_adam_steps_z needs the pass totals {L1, Z, kept}");
  return adam_steps_impl(g, q, params, adam_m, adam_v, t0, n_steps, lr, beta1, beta2, eps, 0.0,
                         flag, use_graph, scratch, scratch_bytes, stream, false, nullptr, nullptr,
                         nullptr, totals);
}

int fm_epi_adam_steps_nccl(const fm_pair_graph* g, const fm_quad_model* q, double* params,
                           double* adam_m, double* adam_v, int64_t t0, int32_t n_steps, double lr,
                           double beta1, double beta2, double eps, double scale, int32_t* flag,
                           void* nccl_comm, double* grad_buf, int32_t use_graph, void* scratch,
                           size_t scratch_bytes, void* stream) {
  FM_REQUIRE(grad_buf, "fm_epi_adam_steps_nccl needs grad_buf [9N + C + 1]");
  return adam_steps_impl(g, q, params, adam_m, adam_v, t0, n_steps, lr, beta1, beta2, eps, scale,
                         flag, use_graph, scratch, scratch_bytes, stream, true, nccl_comm, grad_buf);
}

size_t fm_peer_part_len(const fm_pair_graph* g) {
  if (!g) return 0;
  const int img_blocks = (int)ceil_div((int64_t)g->n_images * 32, kReduceBlock);
  const int n_logical = img_blocks + (cams_by_block(*g) ? (int)ceil_div(g->n_cameras, 2) : 0);
  return (size_t)9 * g->n_images + (g->refine_focal ? g->n_cameras : 0) + (size_t)n_logical;
}

size_t fm_peer_flag_len(const fm_pair_graph* g) {
  if (!g) return 0;
  const int img_blocks = (int)ceil_div((int64_t)g->n_images * 32, kReduceBlock);
  return (size_t)img_blocks + (cams_by_block(*g) ? (size_t)ceil_div(g->n_cameras, 2) : 0);
}

int fm_epi_adam_steps_peer(const fm_pair_graph* g, const fm_quad_model* q, double* params,
                           double* adam_m, double* adam_v, int64_t t0, int32_t n_steps, double lr,
                           double beta1, double beta2, double eps, double scale, int32_t* flag,
                           const fm_peer_group* group, int32_t use_graph, void* scratch,
                           size_t scratch_bytes, void* stream) {
  FM_REQUIRE(group && group->part && group->ready && group->n_ranks >= 1 &&
                 group->rank >= 0 && group->rank < group->n_ranks && group->epoch >= 0,
             "bad peer group");
  FM_REQUIRE(g && (!g->refine_focal || cams_by_block(*g)),
             "the peer-exchange step handles at most %d refined cameras", kBlockCams);
  return adam_steps_impl(g, q, params, adam_m, adam_v, t0, n_steps, lr, beta1, beta2, eps, scale,
                         flag, use_graph, scratch, scratch_bytes, stream, false, nullptr, nullptr, group);
}

void fm_release_cached_graphs(void) {
  std::lock_guard<std::mutex> lk(g_graph_mu);
  for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second);
  g_graphs.clear();
}

}  // extern "C"
