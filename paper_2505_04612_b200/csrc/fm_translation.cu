// Global translation alignment: the per-edge L1 direction loss, its gradient
// and Adam, for B independent random initialisations in lock-step, plus the
// multi-init merge (ref/translation.py:112-186).
//
// Bitwise the reference.  Every floating-point operation is the one numpy
// performs, in numpy's order (explicit _rn intrinsics, so nvcc cannot
// contract a product into an FMA):
//   * per edge, with the reference's orientation delta = c_j - c_i:
//     |delta| = sqrt((d0^2 + d1^2) + d2^2) (np.linalg.norm along axis 1),
//     u = delta / max(|delta|, 1e-8), r = u - d, g_u = sign(r) / m,
//     s = (u0 g0 + u1 g1) + u2 g2, g_delta = (g_u - u s) / |delta|
//     (ref/translation.py:114-121);
//   * per node, the np.add.at scatter order (ref/translation.py:123-124): a
//     left fold starting at 0.0 over the edges where the node is j (ascending
//     edge id, +g_delta), then over the edges where it is i (-g_delta).  The
//     node incidence list is sorted that way (j-side block, then i-side block,
//     each by edge), so the fold is the incidence order;
//   * the loss, np.abs(r).sum() / m, is numpy's pairwise summation over the
//     flattened (m, 3) array (tr_loss_* kernels; the leaf list comes from the
//     host), evaluated once at the state the reference returns it for;
//   * Adam in the numpy expression order with the host's pow() bias
//     corrections (ref/optim.py:30-34).
// So a run's trajectory depends on nothing but its start: identical to the
// reference's for the same seed, in any batch.
//
// Node-centric and deterministic: a warp owns (node v, group of <= 4 runs) and
// gathers the node's incident edges, evaluating each edge once per endpoint
// instead of scattering with atomics.  One read of an edge's direction serves
// all runs of the group; the centres of all runs of a node are contiguous
// ([n][B][3]) so the gather of the other endpoint is one 24R-byte segment.  The
// new centres go to a ping-pong buffer, so one launch is one full optimizer
// step (the fused loss + grad + Adam of ref/translation.py:146-151).
#include <map>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstring>
#include <cstdlib>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kGraphSteps = 200;  // steps per captured CUDA graph (even: keeps ping-pong parity)
constexpr int kPwBlock = 128;     // numpy PW_BLOCKSIZE (pairwise-summation leaf size)

struct TrScratch {
  double4* rec;    // [2m] incidence records {direction, (other node) | side << 31}
  double* buf;     // [n][B][3] ping-pong partner of the caller's centres
  double* m;       // [n][B][3]
  double* v;       // [n][B][3]
  double* lpart;   // [n][B] per-node loss partials (finiteness check)
  const double** ctrl;  // [2] bias-correction tables (1 - b1^t, 1 - b2^t) of the current chunk
  double* cA;      // [n][B][3] ping buffer (the caller's centres are copied in and out)
  double* res;     // [n][B] node residuals (merge)
  int64_t* leaf;   // [n_leaves + 1] pairwise-summation leaf offsets over 3m
  double* lsum;    // [B][n_leaves] leaf sums
};

int64_t max_leaves(int64_t m) { return 3 * m / 32 + 16; }

size_t tr_need(int32_t n, int64_t m, int32_t B) {
  const size_t nb3 = (size_t)n * B * 3;
  const size_t L = (size_t)max_leaves(m);
  return scratch_round((size_t)2 * m * sizeof(double4)) +
         3 * scratch_round(nb3 * sizeof(double)) + 2 * scratch_round((size_t)n * B * sizeof(double)) +
         scratch_round(2 * sizeof(double*)) + scratch_round(nb3 * sizeof(double)) +
         scratch_round((L + 1) * sizeof(int64_t)) +
         scratch_round(L * B * sizeof(double)) + 256;
}

bool tr_carve(int32_t n, int64_t m, int32_t B, void* p, size_t bytes, TrScratch& s) {
  Scratch sc(p, bytes);
  const size_t nb3 = (size_t)n * B * 3;
  const size_t L = (size_t)max_leaves(m);
  s.rec = sc.take<double4>((size_t)2 * m);
  s.buf = sc.take<double>(nb3);
  s.m = sc.take<double>(nb3);
  s.v = sc.take<double>(nb3);
  s.lpart = sc.take<double>((size_t)n * B);
  s.ctrl = sc.take<const double*>(2);
  s.cA = sc.take<double>(nb3);
  s.res = sc.take<double>((size_t)n * B);
  s.leaf = sc.take<int64_t>(L + 1);
  s.lsum = sc.take<double>(L * B);
  return p != nullptr && sc.ok();
}

// numpy's pairwise-summation tree over n elements (pairwise_sum in
// numpy/_core/src/umath/loops_utils.h): leaves of <= 128 elements, a node of
// n > 128 splits at n2 = n/2 rounded down to a multiple of 8.  Host side:
// the leaf offsets, left to right.
void pw_leaves(int64_t lo, int64_t n, std::vector<int64_t>& off) {
  if (n <= kPwBlock) {
    off.push_back(lo + n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pw_leaves(lo, n2, off);
  pw_leaves(lo + n2, n - n2, off);
}

// numpy's leaf sum: < 8 elements a plain left fold from 0.0; otherwise eight
// interleaved accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// then the remainder folded in.
template <typename F>
__device__ double pw_leaf_sum(int64_t lo, int64_t n, F x) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, x(lo + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = x(lo + j);
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x(lo + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, x(lo + i));
  return res;
}

// The tree above evaluated without recursion (no device stack growth):
// post-order walk with an explicit stack; leaf(lo, n) gives a leaf's sum,
// children are added left + right as numpy does.
template <typename Leaf>
__device__ double pw_tree(int64_t n, Leaf leaf) {
  int64_t lo_s[64], n_s[64];
  int stage[64];
  double left[64];
  int sp = 0;
  lo_s[0] = 0, n_s[0] = n, stage[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    const int64_t lo = lo_s[sp], cn = n_s[sp];
    if (cn <= kPwBlock) {
      ret = leaf(lo, cn);
      --sp;
      continue;
    }
    int64_t n2 = cn / 2;
    n2 -= n2 % 8;
    if (stage[sp] == 0) {
      stage[sp] = 1;
      ++sp;
      lo_s[sp] = lo, n_s[sp] = n2, stage[sp] = 0;
    } else if (stage[sp] == 1) {
      left[sp] = ret;
      stage[sp] = 2;
      ++sp;
      lo_s[sp] = lo + n2, n_s[sp] = cn - n2, stage[sp] = 0;
    } else {
      ret = __dadd_rn(left[sp], ret);
      --sp;
    }
  }
  return ret;
}

// Combine from precomputed leaf sums (leaves are visited left to right).
__device__ double pw_combine(int64_t n, const double* leaf_sum) {
  int64_t k = 0;
  return pw_tree(n, [&](int64_t, int64_t) { return leaf_sum[k++]; });
}

// Whole pairwise sum by one thread (small n: the canonicalize norms).
template <typename F>
__device__ double pw_sum(int64_t n, F x) {
  return pw_tree(n, [&](int64_t lo, int64_t cn) { return pw_leaf_sum(lo, cn, x); });
}

// np.linalg.norm of a 3-vector along axis 1: sqrt((x0^2 + x1^2) + x2^2)
__device__ __forceinline__ double norm3(const double d[3]) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                              __dmul_rn(d[2], d[2])));
}

// np.maximum(x, 1e-8): NaN propagates
__device__ __forceinline__ double clamp_len(double x) { return x < 1e-8 ? 1e-8 : x; }

// a / b correctly rounded (bitwise __ddiv_rn) from y = RN(1/b), for the six
// divisions by the same edge length: q0 = RN(a y) is within 1.5 ulp, one
// FMA-residual correction brings it within 1 ulp, and the second is exact
// by Markstein's theorem (y correctly rounded, q within 1 ulp; the residual
// a - b q is exact in an FMA).  The theorem assumes no underflow and finite
// operands: edge_term checks its six quotients once and redoes them with
// __ddiv_rn otherwise (never on real data; kept off the fast path).
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q0 = __dmul_rn(a, y);
  const double q1 = __fma_rn(__fma_rn(-q0, b, a), y, q0);
  return __fma_rn(__fma_rn(-q1, b, a), y, q1);
}

__device__ __forceinline__ bool rcp_div_safe(double q) { return fabs(q) >= 0x1p-960 || q == 0.0; }

// sign(r) / m for the reference's np.sign(r) / m: +-(1/m) (rounded once, as
// the reference's division of +-1 by m), 0 for +-0, NaN for NaN
// (kNaN = false: NaN residuals need not propagate -- the descent's loss
// check raises for them before the gradient is used)
template <bool kNaN>
__device__ __forceinline__ double sign_over_m(double r, double inv_m) {
  const long long bits = __double_as_longlong(r);
  const double sg = __longlong_as_double(__double_as_longlong(inv_m) | (bits & (1ll << 63)));
  if (!kNaN) return r == 0.0 ? 0.0 : sg;
  return r == 0.0 ? 0.0 : (r != r ? r : sg);
}

// One edge in the reference's arithmetic: u = delta / len, r = u - d and
// g_delta (ref/translation.py:114-121); delta = c_j - c_i.
struct EdgeTerm {
  double r[3];
  double gd[3];
};

template <bool kNaN>
__device__ __forceinline__ EdgeTerm edge_term(const double delta[3], const double dir[3],
                                              double inv_m) {
  const double len = clamp_len(norm3(delta));
  const double y = __drcp_rn(len);
  double u[3], gu[3], num[3];
  EdgeTerm t;
#pragma unroll
  for (int k = 0; k < 3; ++k) u[k] = div_rcp(delta[k], len, y);
  bool ok = rcp_div_safe(u[0]) && rcp_div_safe(u[1]) && rcp_div_safe(u[2]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    t.r[k] = __dsub_rn(u[k], dir[k]);
    gu[k] = sign_over_m<kNaN>(t.r[k], inv_m);
  }
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(u[0], gu[0]), __dmul_rn(u[1], gu[1])),
                             __dmul_rn(u[2], gu[2]));
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    num[k] = __dsub_rn(gu[k], __dmul_rn(u[k], s));
    t.gd[k] = div_rcp(num[k], len, y);
    ok = ok && rcp_div_safe(t.gd[k]);
  }
  if (__builtin_expect(!ok, 0)) {
    // exact division everywhere (u first: r and gu depend on it)
#pragma unroll
    for (int k = 0; k < 3; ++k) u[k] = __ddiv_rn(delta[k], len);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      t.r[k] = __dsub_rn(u[k], dir[k]);
      gu[k] = sign_over_m<kNaN>(t.r[k], inv_m);
    }
    const double s2 = __dadd_rn(__dadd_rn(__dmul_rn(u[0], gu[0]), __dmul_rn(u[1], gu[1])),
                                __dmul_rn(u[2], gu[2]));
#pragma unroll
    for (int k = 0; k < 3; ++k) t.gd[k] = __ddiv_rn(__dsub_rn(gu[k], __dmul_rn(u[k], s2)), len);
  }
  return t;
}

enum TrMode { kTrAdam = 0, kTrGrad = 1 };

// Incidence records in node-incidence order: the edge's direction and the
// other endpoint (bit 31: v is the edge's j), so a step gathers one 32-byte
// record per incidence instead of chasing incidence -> edge -> endpoints.
__global__ void tr_incidence_kernel(const fm_dir_graph g, double4* __restrict__ rec) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 2 * g.n_edges) return;
  const int inc = g.node_inc[e];
  const int64_t edge = inc >> 1;
  const int side = inc & 1;  // 0: v is i, 1: v is j
  const int o = side ? g.edge_i[edge] : g.edge_j[edge];
  rec[e] = make_double4(g.dirs[3 * edge], g.dirs[3 * edge + 1], g.dirs[3 * edge + 2],
                        __longlong_as_double((long long)(uint32_t)o | ((long long)side << 31)));
}

__device__ __forceinline__ double flip(double x, long long sign_mask) {
  return __longlong_as_double(__double_as_longlong(x) ^ sign_mask);
}

// One warp per (node, group of R runs); lane = R * slot + run: the warp
// walks the node's incidences kIF x 32/R at a time, every lane evaluating
// one (incidence, run) edge term, so the R lanes of an incidence read the
// record once (broadcast) and the R runs' centres of the other endpoint as one
// contiguous 24R-byte segment.  The terms go to a per-warp shared-memory
// tile; then lane 3 rb + k folds component k of run rb over the tile in
// incidence order (the reference's np.add.at order, see the file comment):
// 3R sequential chains per warp, no redundant shuffled folds.
// kTrAdam: Adam step cur -> nxt.  kTrGrad: write the gradient (API).
#ifndef FM_TR_IF
#define FM_TR_IF 4  // incidences in flight per lane (C3: 2 -> 4 took 0.61 -> 0.54 s)
#endif
#ifndef FM_TR_MINB
#define FM_TR_MINB 2  // resident 256-thread blocks per SM (3: register cap 80, spills, no faster)
#endif

// Loads of centres written in the same launch by other blocks (the
// cluster-persistent descent) must come from L2; across launches the
// read-only path is fine.
template <bool COHERENT>
__device__ __forceinline__ double ld_c(const double* p) {
  return COHERENT ? __ldcg(p) : __ldg(p);
}

// One optimizer step of warp work item w = (node, group of R runs): the
// body of tr_step_kernel, shared with the cluster-persistent descent.
template <int MODE, int R, bool COHERENT>
__device__ __forceinline__ void tr_node_step(const fm_dir_graph& g, const double4* __restrict__ rec,
                                             const double* cur, double* nxt, double* __restrict__ am,
                                             double* __restrict__ av, double* __restrict__ lpart, int B,
                                             double lr, double b1, double b2, double eps,
                                             const double* bc1, const double* bc2, int step,
                                             int32_t* flag, int64_t w, double* tile) {
  constexpr int kSlots = 32 / R;
  constexpr int kIF = FM_TR_IF;  // incidences in flight per lane
  const int lane = threadIdx.x & 31;
  const int groups = (B + R - 1) / R;
  if (w >= (int64_t)g.n_nodes * groups) return;
  if (MODE == kTrAdam && (COHERENT ? *(volatile int32_t*)flag : *flag)) return;
  const int v = (int)(w / groups);
  const int rb = lane % R, slot = lane / R;
  const int b = (int)(w % groups) * R + rb;  // this lane's run
  const int bl = b < B ? b : B - 1;           // idle lanes mirror a valid run
  const double inv_m = __ddiv_rn(1.0, (double)g.n_edges);
  // folding role: lane 3 fr + fk folds component fk of run fr of the group
  const int fr = lane / 3, fk = lane - 3 * (lane / 3);
  const bool folder = lane < 3 * R;
  const int fb = (int)(w % groups) * R + fr;

  double cv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) cv[k] = COHERENT ? __ldcg(cur + ((int64_t)v * B + bl) * 3 + k)
                                               : cur[((int64_t)v * B + bl) * 3 + k];
  double acc = 0.0, lacc = 0.0;
  const int e0 = g.node_off[v], e1 = g.node_off[v + 1];
  for (int base = e0; base < e1; base += kIF * kSlots) {
    double4 r[kIF];
#pragma unroll
    for (int f = 0; f < kIF; ++f) {
      const int e = base + f * kSlots + slot;
      r[f] = rec[e < e1 ? e : e0];
    }
    double c[kIF][3];
#pragma unroll
    for (int f = 0; f < kIF; ++f) {
      const double* p = cur + ((int64_t)(__double_as_longlong(r[f].w) & 0x7fffffff) * B + bl) * 3;
#pragma unroll
      for (int k = 0; k < 3; ++k) c[f][k] = ld_c<COHERENT>(p + k);
    }
#pragma unroll
    for (int f = 0; f < kIF; ++f) {
      // v is the edge's j -> delta = c_v - c_o = -(c_o - c_v) (exact), term +g_delta;
      // v is the edge's i -> delta = c_o - c_v, term -g_delta (np.add.at(i, -))
      const long long vj = (__double_as_longlong(r[f].w) >> 31) & 1;
      const long long to_delta = vj << 63, to_term = (vj ^ 1) << 63;
      double delta[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) delta[k] = flip(__dsub_rn(c[f][k], cv[k]), to_delta);
      const double dir[3] = {r[f].x, r[f].y, r[f].z};
      const EdgeTerm t = edge_term<MODE == kTrGrad>(delta, dir, inv_m);
      const bool live = base + f * kSlots + slot < e1;
      // past the node's last incidence: -0.0, the exact identity of the fold
#pragma unroll
      for (int k = 0; k < 3; ++k) tile[(f * 32 + lane) * 3 + k] = live ? flip(t.gd[k], to_term) : -0.0;
      if (!vj && live) lacc += fabs(t.r[0]) + fabs(t.r[1]) + fabs(t.r[2]);
    }
    __syncwarp();
    if (folder) {
      // incidence base + q (q = f kSlots + s) of run fr sits at
      // [(f 32 + s R + fr) 3 + fk] = [q 3R + lane]
#pragma unroll
      for (int q = 0; q < kIF * kSlots; ++q) acc = __dadd_rn(acc, tile[q * 3 * R + lane]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int off = R; off < 32; off <<= 1) lacc += __shfl_xor_sync(0xffffffffu, lacc, off);
  lacc = __shfl_sync(0xffffffffu, lacc, fr < R ? fr : 0);  // run fr's loss partial
  if (!folder || fb >= B) return;
  const int64_t base = ((int64_t)v * B + fb) * 3;
  if (fk == 0) lpart[(int64_t)v * B + fb] = lacc;
  if (MODE == kTrGrad) {
    nxt[base + fk] = acc;
    return;
  }
  if (!isfinite(lacc)) {
    atomicMax(flag, FM_ERR_NONFINITE_TRANSLATION);
    return;
  }
  if (!isfinite(acc)) {
    atomicMax(flag, FM_ERR_NONFINITE_GRAD);
    return;
  }
  const double c1 = bc1[step], c2 = bc2[step];
  const double ck = COHERENT ? __ldcg(cur + base + fk) : cur[base + fk];
  const double mk = __dadd_rn(__dmul_rn(b1, am[base + fk]), __dmul_rn(1.0 - b1, acc));
  const double vk = __dadd_rn(__dmul_rn(b2, av[base + fk]), __dmul_rn(1.0 - b2, __dmul_rn(acc, acc)));
  am[base + fk] = mk;
  av[base + fk] = vk;
  nxt[base + fk] = __dsub_rn(ck, __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, c1)),
                                           __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, c2)), eps)));
}

constexpr int kTrTile = FM_TR_IF * 32 * 3;  // doubles per warp: [kIF * kSlots][R][3]

template <int MODE, int R>
__global__ void __launch_bounds__(256, FM_TR_MINB) tr_step_kernel(const fm_dir_graph g, const double4* __restrict__ rec,
                               const double* __restrict__ cur,
                               double* __restrict__ nxt, double* __restrict__ am,
                               double* __restrict__ av, double* __restrict__ lpart, int B,
                               double lr, double b1, double b2, double eps,
                               const double* const* __restrict__ bc, int step, int32_t* flag) {
  __shared__ double tile_all[8][kTrTile];
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  tr_node_step<MODE, R, false>(g, rec, cur, nxt, am, av, lpart, B, lr, b1, b2, eps,
                               MODE == kTrAdam ? bc[0] : nullptr, MODE == kTrAdam ? bc[1] : nullptr,
                               step, flag, w, tile_all[threadIdx.x >> 5]);
}

// Small graphs (<= 2 warp work items per warp of one cluster: config 1, the acceptance
// scenes): the whole descent in ONE launch of one thread-block cluster --
// every step the warps run their work items (tr_node_step, the same
// arithmetic as the per-step kernel), then the cluster barrier (release /
// acquire at cluster scope) publishes the new centres to the other blocks;
// centres written in the launch are read from L2 (ld.cg).  Replaces one
// graph-replayed launch per step (launch + drain latency dominated at these
// sizes).  Every thread runs every step and every barrier: a raised flag
// turns the remaining steps into no-ops instead of an early exit.
constexpr int kClusterMax = 8;  // blocks per cluster (portable size; 16 is tried first)

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int R>
__global__ void __launch_bounds__(256) tr_steps_cluster_kernel(const fm_dir_graph g, const double4* __restrict__ rec,
                                                           double* c0, double* c1, double* __restrict__ am,
                                                           double* __restrict__ av, double* __restrict__ lpart,
                                                           int B, double lr, double b1, double b2, double eps,
                                                           const double* bc1, const double* bc2, int steps,
                                                           int32_t* flag) {
  __shared__ double tile_all[8][kTrTile];
  const int groups = (B + R - 1) / R;
  const int64_t n_work = (int64_t)g.n_nodes * groups;
  const int64_t stride = (int64_t)gridDim.x * 8;
  double* tile = tile_all[threadIdx.x >> 5];
  for (int k = 0; k < steps; ++k) {
    const double* cur = (k & 1) ? c1 : c0;
    double* nxt = (k & 1) ? c0 : c1;
    for (int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); w < n_work; w += stride)
      tr_node_step<kTrAdam, R, true>(g, rec, cur, nxt, am, av, lpart, B, lr, b1, b2, eps, bc1, bc2, k,
                                     flag, w, tile);
    cluster_sync_all();
  }
}

// |r| of flattened element q of the (m, 3) residual array of run b
__device__ __forceinline__ double abs_residual(const fm_dir_graph& g, const double* __restrict__ c,
                                               int B, int b, int64_t q) {
  const int64_t e = q / 3;
  const int k = (int)(q - 3 * e);
  const int i = g.edge_i[e], j = g.edge_j[e];
  double ci[3], cj[3], delta[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ci[a] = c[((int64_t)i * B + b) * 3 + a];
    cj[a] = c[((int64_t)j * B + b) * 3 + a];
    delta[a] = __dsub_rn(cj[a], ci[a]);
  }
  const double len = clamp_len(norm3(delta));
  return fabs(__dsub_rn(__ddiv_rn(delta[k], len), g.dirs[3 * e + k]));
}

// loss = np.abs(r).sum() / m (ref/translation.py:119): pairwise leaves
// (thread per (leaf, run)), then the combine (thread per run).
__global__ void tr_loss_leaf_kernel(const fm_dir_graph g, const double* __restrict__ c, int B,
                                    const int64_t* __restrict__ leaf, int64_t n_leaves,
                                    double* __restrict__ lsum) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (l >= n_leaves) return;
  const int64_t lo = l ? leaf[l - 1] : 0;
  lsum[(int64_t)b * n_leaves + l] =
      pw_leaf_sum(lo, leaf[l] - lo, [&](int64_t q) { return abs_residual(g, c, B, b, q); });
}

__global__ void tr_loss_combine_kernel(int64_t n_elem, const double* __restrict__ lsum,
                                       int64_t n_leaves, int64_t m, double* __restrict__ loss) {
  const int b = blockIdx.x;
  loss[b] = __ddiv_rn(pw_combine(n_elem, lsum + (int64_t)b * n_leaves), (double)m);
}

// canonicalize (ref/translation.py:128-134), block per run, in place:
// mean over axis 0 is numpy's sequential row accumulation, the mean norm a
// pairwise sum.
__global__ void tr_canon_kernel(double* __restrict__ c, int n, int B) {
  __shared__ double mean[3];
  __shared__ double scale;
  const int b = blockIdx.x;
  if (threadIdx.x < 3) {
    const int k = threadIdx.x;
    double s = c[(int64_t)b * 3 + k];
    for (int v = 1; v < n; ++v) s = __dadd_rn(s, c[((int64_t)v * B + b) * 3 + k]);
    mean[k] = __ddiv_rn(s, (double)n);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double mu[3] = {mean[0], mean[1], mean[2]};
    const double tot = pw_sum(n, [&](int64_t v) {
      double o[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) o[k] = __dsub_rn(c[(v * B + b) * 3 + k], mu[k]);
      return norm3(o);
    });
    scale = __ddiv_rn(tot, (double)n);
  }
  __syncthreads();
  const double sc = scale;
  for (int v = threadIdx.x; v < n; v += blockDim.x)
    for (int k = 0; k < 3; ++k) {
      double x = __dsub_rn(c[((int64_t)v * B + b) * 3 + k], mean[k]);
      if (sc > 1e-8) x = __ddiv_rn(x, sc);
      c[((int64_t)v * B + b) * 3 + k] = x;
    }
}

// per_node_residuals (ref/translation.py:155-166), warp per (node, run):
// the np.add.at order is the edges where the node is i (the second block of
// its incidence list), then those where it is j (the first block).
__global__ void tr_node_res_kernel(const fm_dir_graph g, const double* __restrict__ c, int B,
                                   double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= (int64_t)g.n_nodes * B) return;
  const int v = (int)(w / B), b = (int)(w % B);
  const int e0 = g.node_off[v], e1 = g.node_off[v + 1];
  // first i-side incidence (side bit 0)
  int mid = e1;
  for (int e = e0; e < e1; e += 32) {
    const bool is_i = e + lane < e1 && !(g.node_inc[e + lane] & 1);
    const unsigned m = __ballot_sync(0xffffffffu, is_i);
    if (m) {
      mid = e + __ffs(m) - 1;
      break;
    }
  }
  double acc = 0.0;
  for (int part = 0; part < 2; ++part) {
    const int lo = part ? e0 : mid, hi = part ? mid : e1;
    for (int e = lo; e < hi; e += 32) {
      double r = 0.0;
      if (e + lane < hi) {
        const int64_t edge = g.node_inc[e + lane] >> 1;
        const int i = g.edge_i[edge], j = g.edge_j[edge];
        double delta[3];
        for (int k = 0; k < 3; ++k)
          delta[k] = __dsub_rn(c[((int64_t)j * B + b) * 3 + k], c[((int64_t)i * B + b) * 3 + k]);
        const double len = clamp_len(norm3(delta));
        double a[3];
        for (int k = 0; k < 3; ++k) a[k] = fabs(__dsub_rn(__ddiv_rn(delta[k], len), g.dirs[3 * edge + k]));
        r = __dadd_rn(__dadd_rn(a[0], a[1]), a[2]);
      }
      const int cnt = min(32, hi - e);
      for (int s = 0; s < cnt; ++s) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, r, s));
    }
  }
  if (lane == 0) out[(int64_t)v * B + b] = __ddiv_rn(acc, fmax((double)(e1 - e0), 1.0));
}

// per-node argmin over runs (first minimum, as np.argmin) + gather
__global__ void tr_merge_kernel(const double* __restrict__ c, const double* __restrict__ res, int n,
                                int B, double* __restrict__ merged, int32_t* __restrict__ choice) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  int best = 0;
  double bv = res[(int64_t)v * B];
  for (int b = 1; b < B; ++b) {
    const double x = res[(int64_t)v * B + b];
    if (isnan(bv)) break;
    if (x < bv || isnan(x)) {
      bv = x;
      best = b;
    }
  }
  if (choice) choice[v] = best;
  for (int k = 0; k < 3; ++k) merged[3 * v + k] = c[((int64_t)v * B + best) * 3 + k];
}

int check_dir_graph(const fm_dir_graph* g, int32_t B) {
  FM_REQUIRE(g, "null direction graph");
  FM_REQUIRE(g->n_nodes >= 0 && g->n_edges >= 0, "negative graph size");
  FM_REQUIRE(B >= 1, "need at least one run");
  return FM_OK;
}

unsigned warp_blocks(int64_t warps) { return (unsigned)ceil_div(warps * 32, 256); }

// runs per warp: 4 for every batch (idle lanes when B % 4 != 0), 1 for a
// single run.  The arithmetic of a run does not depend on R (the fold is in
// incidence order), so the grouping is a pure throughput choice.
int run_group(int B) {
  if (const char* env = getenv("FM_TR_R")) return B >= 2 ? atoi(env) : 1;  // tuning override
  return B >= 2 ? 4 : 1;
}

int build_incidence(const fm_dir_graph& g, const TrScratch& s, cudaStream_t st) {
  if (g.n_edges == 0) return FM_OK;
  tr_incidence_kernel<<<(unsigned)ceil_div(2 * g.n_edges, 256), 256, 0, st>>>(g, s.rec);
  FM_LAUNCHED(tr_incidence_kernel);
  return FM_OK;
}

int enqueue_tr_steps(const fm_dir_graph& g, double* c0, double* c1, const TrScratch& s, int B,
                     int steps, double lr, double b1, double b2, double eps, int32_t* flag,
                     cudaStream_t st) {
  const int R = run_group(B);
  const unsigned blocks = warp_blocks((int64_t)g.n_nodes * ((B + R - 1) / R));
  for (int k = 0; k < steps; ++k) {
    const double* cur = (k & 1) ? c1 : c0;
    double* nxt = (k & 1) ? c0 : c1;
    if (R == 1)
      tr_step_kernel<kTrAdam, 1><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.ctrl, k, flag);
    else if (R == 2)
      tr_step_kernel<kTrAdam, 2><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.ctrl, k, flag);
    else if (R == 8)
      tr_step_kernel<kTrAdam, 8><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.ctrl, k, flag);
    else
      tr_step_kernel<kTrAdam, 4><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.ctrl, k, flag);
    FM_LAUNCHED(tr_step_kernel);
  }
  return FM_OK;
}

__global__ void tr_set_ctrl_kernel(const double** ctrl, const double* c1, const double* c2) {
  ctrl[0] = c1;
  ctrl[1] = c2;
}

// loss_out[b] = np.abs(r).sum() / m at centres c (ref/translation.py:119),
// numpy's pairwise summation over the flattened (m, 3) residuals
int enqueue_exact_loss(const fm_dir_graph& g, const double* c, int B, const TrScratch& s,
                       double* loss_out, cudaStream_t st) {
  const int64_t n_elem = 3 * g.n_edges;
  std::vector<int64_t> off;
  pw_leaves(0, n_elem, off);
  const int64_t L = (int64_t)off.size();
  FM_REQUIRE(L <= max_leaves(g.n_edges), "pairwise leaf bound");
  FM_CUDA(cudaMemcpyAsync(s.leaf, off.data(), L * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  // the host vector must outlive the copy: pageable memcpy is staged synchronously
  tr_loss_leaf_kernel<<<dim3((unsigned)ceil_div(L, 128), (unsigned)B), 128, 0, st>>>(g, c, B, s.leaf, L,
                                                                                    s.lsum);
  FM_LAUNCHED(tr_loss_leaf_kernel);
  tr_loss_combine_kernel<<<B, 1, 0, st>>>(n_elem, s.lsum, L, g.n_edges, loss_out);
  FM_LAUNCHED(tr_loss_combine_kernel);
  return FM_OK;
}

template <int R>
cudaError_t launch_tr_cluster_r(const fm_dir_graph& g, const TrScratch& s, int B, int steps, double lr,
                                double b1, double b2, double eps, const double* table, int32_t* flag,
                                int nblk, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nblk);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)nblk;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (nblk > kClusterMax) {
    cudaError_t e = cudaFuncSetAttribute(tr_steps_cluster_kernel<R>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaLaunchKernelEx(&cfg, tr_steps_cluster_kernel<R>, g, (const double4*)s.rec, s.cA, s.buf, s.m,
                            s.v, s.lpart, B, lr, b1, b2, eps, table, table + steps, steps, flag);
}

// The whole descent as one cluster launch (small graphs); false: not taken
// (too many work items, disabled, or the launch was refused -- the caller
// then replays the per-step graphs).  Measured at config 1 (50 nodes, 3
// runs, 6000 steps; tools/c1_tr_probe.py): per-step graphs 39-45 ms; one
// cluster of 8 blocks, R = 4: 37 ms; 16 blocks (non-portable size), R = 2:
// 29 ms -- twice the warps, so each SM sub-partition hides more latency.
bool launch_tr_cluster(const fm_dir_graph& g, const TrScratch& s, int B, int steps, double lr, double b1,
                       double b2, double eps, const double* table, int32_t* flag, cudaStream_t st) {
  if (getenv("FM_TR_NOCLUSTER")) return false;
  const char* env_r = getenv("FM_TRC_R");  // tuning overrides
  const char* env_c = getenv("FM_TRC_CLUSTER");
  const int R = env_r ? atoi(env_r) : (B >= 2 ? 2 : 1);
  const int64_t n_work = (int64_t)g.n_nodes * ((B + R - 1) / R);
  for (int cmax : {env_c ? atoi(env_c) : 2 * kClusterMax, kClusterMax}) {
    if (n_work > 2 * 8 * (int64_t)cmax) continue;
    const int nblk = (int)std::min<int64_t>(std::max<int64_t>(ceil_div(n_work, 8), 1), cmax);
    cudaError_t e;
    switch (R) {
      case 1: e = launch_tr_cluster_r<1>(g, s, B, steps, lr, b1, b2, eps, table, flag, nblk, st); break;
      case 4: e = launch_tr_cluster_r<4>(g, s, B, steps, lr, b1, b2, eps, table, flag, nblk, st); break;
      case 8: e = launch_tr_cluster_r<8>(g, s, B, steps, lr, b1, b2, eps, table, flag, nblk, st); break;
      default: e = launch_tr_cluster_r<2>(g, s, B, steps, lr, b1, b2, eps, table, flag, nblk, st); break;
    }
    if (e == cudaSuccess) return true;
    cudaGetLastError();  // clear; try the portable size, then fall back
  }
  return false;
}

struct TrKey {
  std::vector<uintptr_t> k;
  bool operator<(const TrKey& o) const { return k < o.k; }
};
std::mutex g_tr_mu;
std::map<TrKey, cudaGraphExec_t> g_tr_graphs;

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_tr_scratch_bytes(int32_t n_nodes, int64_t n_edges, int32_t n_runs) {
  return tr_need(n_nodes, n_edges, n_runs);
}

int fm_tr_loss_grad(const fm_dir_graph* g, const double* centers, int32_t B, double* loss_out,
                    double* grad_out, void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = check_dir_graph(g, B)) return rc;
  TrScratch s;
  FM_REQUIRE(tr_carve(g->n_nodes, g->n_edges, B, scratch, scratch_bytes, s), "translation scratch too small");
  FM_REQUIRE(g->n_edges > 0, "graph has no edges");
  cudaStream_t st = as_stream(stream);
  if (g->n_nodes == 0) return FM_OK;
  if (int rc = build_incidence(*g, s, st)) return rc;
  const int R = run_group(B);
  const unsigned blocks = warp_blocks((int64_t)g->n_nodes * ((B + R - 1) / R));
  if (R == 1)
    tr_step_kernel<kTrGrad, 1><<<blocks, 256, 0, st>>>(*g, s.rec, centers, grad_out, nullptr, nullptr,
                                                       s.lpart, B, 0, 0, 0, 0, nullptr, 0, nullptr);
  else
    tr_step_kernel<kTrGrad, 4><<<blocks, 256, 0, st>>>(*g, s.rec, centers, grad_out, nullptr, nullptr,
                                                       s.lpart, B, 0, 0, 0, 0, nullptr, 0, nullptr);
  FM_LAUNCHED(tr_step_kernel);
  return enqueue_exact_loss(*g, centers, B, s, loss_out, st);
}

int fm_tr_align(const fm_dir_graph* g, double* centers, int32_t B, int32_t steps, double lr,
                double beta1, double beta2, double eps, double* loss_out, int32_t* flag,
                void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = check_dir_graph(g, B)) return rc;
  FM_REQUIRE(flag, "fm_tr_align needs a device flag word");
  FM_REQUIRE(steps >= 0, "negative step count");
  FM_REQUIRE(g->n_edges > 0, "graph has no edges");
  TrScratch s;
  FM_REQUIRE(tr_carve(g->n_nodes, g->n_edges, B, scratch, scratch_bytes, s), "translation scratch too small");
  cudaStream_t st = as_stream(stream);
  const int n = g->n_nodes;
  const size_t nb3 = (size_t)n * B * 3;
  if (n == 0 || steps == 0) return FM_OK;
  FM_CUDA(cudaMemsetAsync(s.m, 0, nb3 * sizeof(double), st));
  FM_CUDA(cudaMemsetAsync(s.v, 0, nb3 * sizeof(double), st));
  if (int rc = build_incidence(*g, s, st)) return rc;
  // bias corrections 1 - beta^t of every step with the host's pow (the
  // reference's Python `beta ** t`), one stream-ordered table per call
  std::vector<double> bc(2 * (size_t)steps);
  for (int k = 0; k < steps; ++k) {
    bc[k] = 1.0 - pow(beta1, (double)(k + 1));
    bc[steps + k] = 1.0 - pow(beta2, (double)(k + 1));
  }
  double* table = nullptr;
  FM_CUDA(cudaMallocAsync(&table, bc.size() * sizeof(double), st));
  FM_CUDA(cudaMemcpyAsync(table, bc.data(), bc.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  // the descent ping-pongs between two scratch buffers, so the captured
  // graphs depend only on the scratch / graph pointers and are reused
  // across calls
  FM_CUDA(cudaMemcpyAsync(s.cA, centers, nb3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  int done = launch_tr_cluster(*g, s, B, steps, lr, beta1, beta2, eps, table, flag, st) ? steps : 0;
  while (done < steps) {
    const int chunk = std::min(kGraphSteps, steps - done);
    tr_set_ctrl_kernel<<<1, 1, 0, st>>>(s.ctrl, table + done, table + steps + done);
    FM_LAUNCHED(tr_set_ctrl_kernel);
    if (chunk == kGraphSteps) {
      TrKey key;
      for (const void* p : {(const void*)g->edge_i, (const void*)g->edge_j, (const void*)g->dirs,
                            (const void*)g->node_off, (const void*)g->node_inc, (const void*)s.rec,
                            (const void*)s.cA, (const void*)s.buf, (const void*)s.m, (const void*)s.v,
                            (const void*)s.lpart, (const void*)s.ctrl, (const void*)flag})
        key.k.push_back(reinterpret_cast<uintptr_t>(p));
      key.k.push_back((uintptr_t)n);
      key.k.push_back((uintptr_t)g->n_edges);
      key.k.push_back((uintptr_t)B);
      for (double d : {lr, beta1, beta2, eps}) {
        uintptr_t u;
        memcpy(&u, &d, sizeof(u));
        key.k.push_back(u);
      }
      cudaGraphExec_t exec = nullptr;
      {
        std::lock_guard<std::mutex> lk(g_tr_mu);
        auto it = g_tr_graphs.find(key);
        if (it != g_tr_graphs.end()) exec = it->second;
      }
      if (!exec) {
        cudaStream_t cs;
        FM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FM_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_tr_steps(*g, s.cA, s.buf, s, B, chunk, lr, beta1, beta2, eps, flag, cs);
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
        std::lock_guard<std::mutex> lk(g_tr_mu);
        if (g_tr_graphs.size() >= 16) {
          for (auto& kv : g_tr_graphs) cudaGraphExecDestroy(kv.second);
          g_tr_graphs.clear();
        }
        g_tr_graphs[key] = exec;
      }
      FM_CUDA(cudaGraphLaunch(exec, st));
    } else {
      if (int rc = enqueue_tr_steps(*g, s.cA, s.buf, s, B, chunk, lr, beta1, beta2, eps, flag, st))
        return rc;
    }
    done += chunk;
  }
  // step k reads cA (k even) or buf: an odd step count ends in buf (full
  // graph chunks are even).  The reference returns the loss evaluated at the
  // last step, i.e. before its update.
  const bool odd = steps & 1;
  const double* fin = odd ? s.buf : s.cA;
  const double* pre = odd ? s.cA : s.buf;
  if (int rc = enqueue_exact_loss(*g, pre, B, s, loss_out, st)) return rc;
  FM_CUDA(cudaMemcpyAsync(centers, fin, nb3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  FM_CUDA(cudaFreeAsync(table, st));
  return FM_OK;
}

int fm_tr_canonicalize(double* centers, int32_t n_nodes, int32_t B, void* scratch,
                       size_t scratch_bytes, void* stream) {
  (void)scratch;
  (void)scratch_bytes;
  FM_REQUIRE(n_nodes >= 0 && B >= 1, "bad canonicalize sizes");
  if (n_nodes == 0) return FM_OK;
  tr_canon_kernel<<<B, 256, 0, as_stream(stream)>>>(centers, n_nodes, B);
  FM_LAUNCHED(tr_canon_kernel);
  return FM_OK;
}

int fm_tr_node_residuals(const fm_dir_graph* g, const double* centers, int32_t B, double* out,
                         void* stream) {
  if (int rc = check_dir_graph(g, B)) return rc;
  if (g->n_nodes == 0) return FM_OK;
  tr_node_res_kernel<<<warp_blocks((int64_t)g->n_nodes * B), 256, 0, as_stream(stream)>>>(*g, centers, B, out);
  FM_LAUNCHED(tr_node_res_kernel);
  return FM_OK;
}

int fm_tr_merge(const fm_dir_graph* g, double* centers, int32_t B, double* merged, int32_t* choice,
                void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = check_dir_graph(g, B)) return rc;
  TrScratch s;
  FM_REQUIRE(tr_carve(g->n_nodes, g->n_edges, B, scratch, scratch_bytes, s), "translation scratch too small");
  cudaStream_t st = as_stream(stream);
  const int n = g->n_nodes;
  if (n == 0) return FM_OK;
  tr_canon_kernel<<<B, 256, 0, st>>>(centers, n, B);
  FM_LAUNCHED(tr_canon_kernel);
  tr_node_res_kernel<<<warp_blocks((int64_t)n * B), 256, 0, st>>>(*g, centers, B, s.res);
  FM_LAUNCHED(tr_node_res_kernel);
  tr_merge_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(centers, s.res, n, B, merged, choice);
  FM_LAUNCHED(tr_merge_kernel);
  return FM_OK;
}

}  // extern "C"
