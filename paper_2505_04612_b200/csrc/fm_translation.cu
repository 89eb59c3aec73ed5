// Global translation alignment: the per-edge L1 direction loss, its gradient
// and Adam, for B independent random initialisations in lock-step, plus the
// multi-init merge (ref/translation.py:112-186).
//
// Node-centric and deterministic: a warp owns (node v, group of <= 4 runs) and
// gathers the node's incident edges (fixed lane-strided order + fixed warp
// butterfly), evaluating each edge once per endpoint instead of scattering with
// atomics.  One read of an edge's direction serves all runs of the group; the
// centres of all runs of a node are contiguous ([n][B][3]) so the gather of
// the other endpoint is one 96-byte segment.  The new centres go to a
// ping-pong buffer, so one launch is one full optimizer step (the fused
// loss + grad + Adam of ref/translation.py:146-151).
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

struct TrScratch {
  double4* rec;   // [2m] incidence records {direction, (other node) | side << 31}
  double* buf;    // [n][B][3] ping-pong partner of the caller's centres
  double* m;      // [n][B][3]
  double* v;      // [n][B][3]
  double* lpart;  // [n][B] per-node loss partials (edges where the node is i)
  double* bc;     // [2][kGraphSteps] bias corrections
  double* res;    // [n][B] node residuals (merge)
};

size_t tr_need(int32_t n, int64_t m, int32_t B) {
  const size_t nb3 = (size_t)n * B * 3;
  return scratch_round((size_t)2 * m * sizeof(double4)) +
         3 * scratch_round(nb3 * sizeof(double)) + 2 * scratch_round((size_t)n * B * sizeof(double)) +
         scratch_round(2 * kGraphSteps * sizeof(double)) + 256;
}

bool tr_carve(int32_t n, int64_t m, int32_t B, void* p, size_t bytes, TrScratch& s) {
  Scratch sc(p, bytes);
  const size_t nb3 = (size_t)n * B * 3;
  s.rec = sc.take<double4>((size_t)2 * m);
  s.buf = sc.take<double>(nb3);
  s.m = sc.take<double>(nb3);
  s.v = sc.take<double>(nb3);
  s.lpart = sc.take<double>((size_t)n * B);
  s.bc = sc.take<double>(2 * kGraphSteps);
  s.res = sc.take<double>((size_t)n * B);
  return p != nullptr && sc.ok();
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// 1/sqrt(q) for normal q > 0: hardware approximation + two Newton steps
// (~1 ulp; no slow-path call)
__device__ __forceinline__ double rsqrt_nr(double q) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  const double h = 0.5 * q;
  y = fma(y, fma(-h * y, y, 0.5), y);
  y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}

// np.sign for finite x on the integer pipe: +-1 with x's sign bit, 0 for +-0
// (a NaN residual yields +-1 here; the NaN loss it comes with raises anyway)
__device__ __forceinline__ double sign_or_zero(double x) {
  const int hi = __double2hiint(x);
  const int one = 0x3FF00000 | (hi & (int)0x80000000);
  return __hiloint2double(x != 0.0 ? one : 0, 0);
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

// One warp per (node, group of R runs); lane = R * slot + run: the warp
// walks the node's incidences 32/R at a time, every lane evaluates one
// (incidence, run) term, so the R lanes of an incidence read the record once
// (broadcast) and the R runs' centres of the other endpoint as one contiguous
// 24R-byte segment.  Two incidences per lane are in flight (the step is a
// chain of dependent L2 gathers).  Fixed-order butterflies over the slots.
// kTrAdam: Adam step cur -> nxt.  kTrGrad: write the gradient (API).
//
// Per term, with e = c_o - c_v, s = +1 if v is the edge's i else -1 and the
// reference's u = s e / |e|, r = u - d, g_u = sign(r) / m
// (ref/translation.py:112-125): writing w = e / |e| and d' = s d,
// r = s (w - d'), so |r| = |w - d'|, sign(r) = s sign(w - d') and the node's
// gradient term -s g_delta = -(sign(w - d') - w (w . sign(w - d'))) / (m |e|)
// carries no sign of its own -- one formula for both endpoints, 1/m once.
template <int MODE, int R>
__global__ void __launch_bounds__(256) tr_step_kernel(const fm_dir_graph g, const double4* __restrict__ rec,
                               const double* __restrict__ cur,
                               double* __restrict__ nxt, double* __restrict__ am,
                               double* __restrict__ av, double* __restrict__ lpart, int B,
                               double lr, double b1, double b2, double eps,
                               const double* __restrict__ bc, int step, int32_t* flag) {
  constexpr int kSlots = 32 / R;
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int groups = (B + R - 1) / R;
  if (w >= (int64_t)g.n_nodes * groups) return;
  if (MODE == kTrAdam && *flag) return;
  const int v = (int)(w / groups);
  const int rb = lane % R, slot = lane / R;
  const int b = (int)(w % groups) * R + rb;  // this lane's run
  const bool run_ok = b < B;
  const int bl = run_ok ? b : B - 1;          // idle lanes mirror a valid run
  const double inv_m = 1.0 / (double)g.n_edges;

  double cv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) cv[k] = cur[((int64_t)v * B + bl) * 3 + k];
  double acc[3] = {0.0, 0.0, 0.0}, lacc = 0.0;
  auto term = [&](const double4 r, const double co[3]) {
    const bool vj = (__double_as_longlong(r.w) >> 31) & 1;  // v is the edge's j
    const double dp[3] = {vj ? -r.x : r.x, vj ? -r.y : r.y, vj ? -r.z : r.z};
    double e[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) e[k] = co[k] - cv[k];
    const double q = e[0] * e[0] + e[1] * e[1] + e[2] * e[2];
    // 1 / max(|e|, 1e-8) as one fp64 reciprocal square root (the reference
    // divides each component by the clamped norm, ref/translation.py:115-121;
    // same value to within an ulp)
    const double inv = q > 1e-16 ? rsqrt_nr(q) : 1e8;
    double wv[3], sg[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      wv[k] = e[k] * inv;
      sg[k] = sign_or_zero(wv[k] - dp[k]);
    }
    const double wg = wv[0] * sg[0] + wv[1] * sg[1] + wv[2] * sg[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) acc[k] -= (sg[k] - wv[k] * wg) * inv;
    if (!vj) lacc += fabs(wv[0] - dp[0]) + fabs(wv[1] - dp[1]) + fabs(wv[2] - dp[2]);
  };
  const int e0 = g.node_off[v], e1 = g.node_off[v + 1];
  constexpr int kIF = 2;  // incidences in flight per lane (4: more registers, half the warps)
  for (int e = e0 + slot; e < e1; e += kIF * kSlots) {
    double4 r[kIF];
#pragma unroll
    for (int f = 0; f < kIF; ++f) r[f] = rec[e + f * kSlots < e1 ? e + f * kSlots : e];
    double c[kIF][3];
#pragma unroll
    for (int f = 0; f < kIF; ++f) {
      const double* p = cur + ((int64_t)(__double_as_longlong(r[f].w) & 0x7fffffff) * B + bl) * 3;
#pragma unroll
      for (int k = 0; k < 3; ++k) c[f][k] = __ldg(p + k);
    }
#pragma unroll
    for (int f = 0; f < kIF; ++f)
      if (e + f * kSlots < e1) term(r[f], c[f]);
  }
#pragma unroll
  for (int off = R; off < 32; off <<= 1) {
    lacc += __shfl_xor_sync(0xffffffffu, lacc, off);
#pragma unroll
    for (int k = 0; k < 3; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
  }
  if (slot != 0 || !run_ok) return;
#pragma unroll
  for (int k = 0; k < 3; ++k) acc[k] *= inv_m;
  const int64_t base = ((int64_t)v * B + b) * 3;
  lpart[(int64_t)v * B + b] = lacc;
  if (MODE == kTrGrad) {
#pragma unroll
    for (int k = 0; k < 3; ++k) nxt[base + k] = acc[k];
    return;
  }
  if (!isfinite(lacc)) {
    atomicMax(flag, FM_ERR_NONFINITE_TRANSLATION);
    return;
  }
  if (!(isfinite(acc[0]) && isfinite(acc[1]) && isfinite(acc[2]))) {
    atomicMax(flag, FM_ERR_NONFINITE_GRAD);
    return;
  }
  const double c1 = bc[step], c2 = bc[kGraphSteps + step];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double gk = acc[k];
    const double mk = __dadd_rn(__dmul_rn(b1, am[base + k]), __dmul_rn(1.0 - b1, gk));
    const double vk = __dadd_rn(__dmul_rn(b2, av[base + k]), __dmul_rn(1.0 - b2, __dmul_rn(gk, gk)));
    am[base + k] = mk;
    av[base + k] = vk;
    nxt[base + k] = __dsub_rn(cv[k], __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, c1)),
                                               __dadd_rn(sqrt(__ddiv_rn(vk, c2)), eps)));
  }
}

// loss[b] = sum_v lpart[v][b] / m  (fixed-order block reduction, block per run)
__global__ void tr_loss_kernel(const double* __restrict__ lpart, int n, int B, int64_t m,
                               double* __restrict__ loss) {
  __shared__ double red[256];
  const int b = blockIdx.x;
  double acc = 0;
  for (int v = threadIdx.x; v < n; v += 256) acc += lpart[(int64_t)v * B + b];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss[b] = red[0] / (double)m;
}

// canonicalize (ref/translation.py:128-134), block per run, in place
__global__ void tr_canon_kernel(double* __restrict__ c, int n, int B) {
  __shared__ double red[256][3];
  const int b = blockIdx.x;
  double s[3] = {0, 0, 0};
  for (int v = threadIdx.x; v < n; v += 256)
    for (int k = 0; k < 3; ++k) s[k] += c[((int64_t)v * B + b) * 3 + k];
  for (int k = 0; k < 3; ++k) red[threadIdx.x][k] = s[k];
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st)
      for (int k = 0; k < 3; ++k) red[threadIdx.x][k] += red[threadIdx.x + st][k];
    __syncthreads();
  }
  const double mean[3] = {red[0][0] / n, red[0][1] / n, red[0][2] / n};
  __syncthreads();
  double ns = 0;
  for (int v = threadIdx.x; v < n; v += 256) {
    double q = 0;
    for (int k = 0; k < 3; ++k) {
      const double x = c[((int64_t)v * B + b) * 3 + k] - mean[k];
      q += x * x;
    }
    ns += sqrt(q);
  }
  red[threadIdx.x][0] = ns;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) red[threadIdx.x][0] += red[threadIdx.x + st][0];
    __syncthreads();
  }
  const double scale = red[0][0] / n;
  for (int v = threadIdx.x; v < n; v += 256)
    for (int k = 0; k < 3; ++k) {
      double x = c[((int64_t)v * B + b) * 3 + k] - mean[k];
      if (scale > 1e-8) x = x / scale;
      c[((int64_t)v * B + b) * 3 + k] = x;
    }
}

// per_node_residuals (ref/translation.py:155-166), warp per (node, run)
__global__ void tr_node_res_kernel(const fm_dir_graph g, const double* __restrict__ c, int B,
                                   double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= (int64_t)g.n_nodes * B) return;
  const int v = (int)(w / B), b = (int)(w % B);
  const int e0 = g.node_off[v], e1 = g.node_off[v + 1];
  double acc = 0;
  for (int e = e0 + lane; e < e1; e += 32) {
    const int64_t edge = g.node_inc[e] >> 1;
    const int i = g.edge_i[edge], j = g.edge_j[edge];
    double delta[3];
    for (int k = 0; k < 3; ++k) delta[k] = c[((int64_t)j * B + b) * 3 + k] - c[((int64_t)i * B + b) * 3 + k];
    const double len = fmax(sqrt(delta[0] * delta[0] + delta[1] * delta[1] + delta[2] * delta[2]), 1e-8);
    for (int k = 0; k < 3; ++k) acc += fabs(delta[k] / len - g.dirs[3 * edge + k]);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[(int64_t)v * B + b] = acc / fmax((double)(e1 - e0), 1.0);
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
// single run.  A run's summation order depends only on R, so a run's
// trajectory is the same in any batch of >= 2 runs -- the multi-init runs
// sharded over ranks reproduce the single-GPU batch bit for bit.
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
                                                         b1, b2, eps, s.bc, k, flag);
    else if (R == 2)
      tr_step_kernel<kTrAdam, 2><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.bc, k, flag);
    else if (R == 8)
      tr_step_kernel<kTrAdam, 8><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.bc, k, flag);
    else
      tr_step_kernel<kTrAdam, 4><<<blocks, 256, 0, st>>>(g, s.rec, cur, nxt, s.m, s.v, s.lpart, B, lr,
                                                         b1, b2, eps, s.bc, k, flag);
    FM_LAUNCHED(tr_step_kernel);
  }
  return FM_OK;
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
  tr_loss_kernel<<<B, 256, 0, st>>>(s.lpart, g->n_nodes, B, g->n_edges, loss_out);
  FM_LAUNCHED(tr_loss_kernel);
  return FM_OK;
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
  std::vector<double> bc(2 * kGraphSteps, 1.0);
  int done = 0;
  // steps in graph-sized chunks; every chunk starts from `centers` (even length)
  while (done < steps) {
    const int chunk = std::min(kGraphSteps, steps - done);
    for (int k = 0; k < chunk; ++k) {
      const double t = (double)(done + k + 1);
      bc[k] = 1.0 - pow(beta1, t);
      bc[kGraphSteps + k] = 1.0 - pow(beta2, t);
    }
    FM_CUDA(cudaMemcpyAsync(s.bc, bc.data(), bc.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    if (chunk == kGraphSteps) {
      TrKey key;
      for (const void* p : {(const void*)g->edge_i, (const void*)g->edge_j, (const void*)g->dirs,
                            (const void*)g->node_off, (const void*)g->node_inc, (const void*)centers,
                            (const void*)s.buf, (const void*)s.m, (const void*)flag})
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
        int rc = enqueue_tr_steps(*g, centers, s.buf, s, B, chunk, lr, beta1, beta2, eps, flag, cs);
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
      if (int rc = enqueue_tr_steps(*g, centers, s.buf, s, B, chunk, lr, beta1, beta2, eps, flag, st))
        return rc;
      if (chunk & 1) FM_CUDA(cudaMemcpyAsync(centers, s.buf, nb3 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    done += chunk;
  }
  tr_loss_kernel<<<B, 256, 0, st>>>(s.lpart, n, B, g->n_edges, loss_out);
  FM_LAUNCHED(tr_loss_kernel);
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
