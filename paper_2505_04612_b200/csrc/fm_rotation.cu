// Rotation refinement (SURVEY 8f "next" #3): Adam on the mean geodesic
// distance over relative-rotation edges in the 6D parameterisation
// (ref/rotation.py:162-230) -- the same edge-gradient + per-node gather +
// Adam shape as the translation step (fm_translation.cu).
//
// Per step, four kernels captured in CUDA graphs of kChunk steps:
//   rot_R_kernel     6D -> R per node (Gram-Schmidt, ref/optim.py:39-59)
//   rot_node_kernel  warp per node: fixed-order gather of its incident edges'
//                    dtr/dR terms (no float atomics), 6D vector-Jacobian
//                    product (rot6d_vjp) -> grad6, per-node loss partial
//   rot_loss_kernel  fixed-order loss sum, history, best-iterate and
//                    early-stop bookkeeping on the device
//   rot_adam_kernel  best-iterate copy (before the update, as the reference
//                    keeps opt.params.copy()) and the Adam update
// Every kernel returns at entry once the run has stopped, so a chunk past
// the stopping step is a no-op; the host reads the stop word once per chunk.
#include <cmath>
#include <vector>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kChunk = 100;       // steps per CUDA graph (= the early-stop window)
constexpr double kAcosClamp = 1.0 - 1e-12;  // ref/rotation.py:159

struct RotState {       // device bookkeeping (ref/rotation.py:208-227)
  double best_loss;
  int32_t stopped;      // 1: no further steps
  int32_t steps;        // losses recorded
  int32_t improved;     // this step's loss < best (copy params before the update)
  int32_t pad;
};

struct RotScratch {
  double* R;      // [n][9]
  double* g6;     // [n][6]
  double* lpart;  // [n]
  double* m;      // [n][6]
  double* v;      // [n][6]
  double* best;   // [n][6]
  double* bc;     // [2][kChunk]
  RotState* st;
};

size_t rot_need(int32_t n) {
  const size_t n6 = (size_t)n * 6;
  return scratch_round((size_t)n * 9 * sizeof(double)) + 4 * scratch_round(n6 * sizeof(double)) +
         scratch_round((size_t)n * sizeof(double)) + scratch_round(2 * kChunk * sizeof(double)) +
         scratch_round(sizeof(RotState)) + 256;
}

bool rot_carve(int32_t n, void* p, size_t bytes, RotScratch& s) {
  Scratch sc(p, bytes);
  const size_t n6 = (size_t)n * 6;
  s.R = sc.take<double>((size_t)n * 9);
  s.g6 = sc.take<double>(n6);
  s.lpart = sc.take<double>((size_t)n);
  s.m = sc.take<double>(n6);
  s.v = sc.take<double>(n6);
  s.best = sc.take<double>(n6);
  s.bc = sc.take<double>(2 * kChunk);
  s.st = sc.take<RotState>(1);
  return p != nullptr && sc.ok();
}

__global__ void rot_R_kernel(const double* __restrict__ p6, int n, double* __restrict__ R,
                             const RotState* st, int32_t* flag) {
  if (st && st->stopped) return;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int rc = rot6d_to_R(p6 + 6 * k, R + 9 * k);
  if (rc) raise_flag(flag, rc);
}

// Warp per node: the node's incident edges in CSR order, lanes strided, a
// fixed butterfly; edge loss counted at its i endpoint.
__global__ void rot_node_kernel(const fm_rot_graph g, const double* __restrict__ p6,
                                const double* __restrict__ R, double* __restrict__ g6,
                                double* __restrict__ lpart, const RotState* st, const int32_t* flag) {
  if ((st && st->stopped) || *flag) return;
  const int lane = threadIdx.x & 31;
  const int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (v >= g.n_nodes) return;
  const double scale_m = 1.0 / (2.0 * (double)g.n_edges);
  double acc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, lacc = 0.0;
  for (int q = g.node_off[v] + lane; q < g.node_off[v + 1]; q += 32) {
    const int inc = g.node_inc[q];
    const int64_t e = inc >> 1;
    const bool vj = inc & 1;
    const double* Ri = R + 9 * (int64_t)g.edge_i[e];
    const double* Rj = R + 9 * (int64_t)g.edge_j[e];
    const double* A = g.rel + 9 * e;
    double T[9];  // target = rel R_i
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) T[r * 3 + c] = A[r * 3] * Ri[c] + A[r * 3 + 1] * Ri[3 + c] + A[r * 3 + 2] * Ri[6 + c];
    double tr = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) tr += Rj[k] * T[k];
    const double u = fmin(fmax((tr - 1.0) / 2.0, -kAcosClamp), kAcosClamp);
    const double scale = -1.0 / sqrt(1.0 - u * u) * scale_m;  // d acos/du / (2m)
    if (vj) {  // d tr / d R_j = rel R_i
#pragma unroll
      for (int k = 0; k < 9; ++k) acc[k] += scale * T[k];
    } else {   // d tr / d R_i = rel^T R_j
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          acc[r * 3 + c] += scale * (A[r] * Rj[c] + A[3 + r] * Rj[3 + c] + A[6 + r] * Rj[6 + c]);
      lacc += acos(u);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lacc += __shfl_xor_sync(0xffffffffu, lacc, off);
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
  }
  if (lane == 0) {
    double out[6];
    rot6d_vjp(p6 + 6 * v, acc, out);
#pragma unroll
    for (int k = 0; k < 6; ++k) g6[6 * v + k] = out[k];
    lpart[v] = lacc;
  }
}

// One block: loss = sum lpart / m in a fixed order; history; best and stop
// rules of ref/rotation.py:217-227.  st == nullptr: loss only (API).
__global__ void rot_loss_kernel(const double* __restrict__ lpart, int n, int64_t m,
                                double* __restrict__ loss_out, double* __restrict__ history,
                                RotState* st, int32_t* flag) {
  if (st && st->stopped) return;
  __shared__ double red[256];
  double a = 0.0;
  for (int v = threadIdx.x; v < n; v += 256) a += lpart[v];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x != 0) return;
  const double loss = red[0] / (double)m;
  if (loss_out) *loss_out = loss;
  if (!st) return;
  if (*flag) {
    st->stopped = 1;
    return;
  }
  if (!isfinite(loss)) {
    raise_flag(flag, FM_ERR_NONFINITE_ROTATION);
    st->stopped = 1;
    return;
  }
  const int step = st->steps;
  history[step] = loss;
  st->steps = step + 1;
  st->improved = loss < st->best_loss;
  if (st->improved) st->best_loss = loss;
  bool stop = loss < 1e-12;
  if (!stop && step >= kChunk) {
    const double prev = history[step - kChunk];
    stop = fabs(prev - loss) < 1e-9 * fmax(prev, 1e-12);
  }
  st->stopped = stop ? 2 : 0;  // 2: stop after this step's best-iterate copy, no update
}

__global__ void rot_adam_kernel(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
                                double* __restrict__ best, const double* __restrict__ g, int64_t n6,
                                double lr, double b1, double b2, double eps,
                                const double* __restrict__ bc, int k, RotState* st, const int32_t* flag) {
  const int32_t stopped = st->stopped;
  if (stopped == 1 || *flag) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n6) {
    if (st->improved) best[q] = p[q];
    if (stopped == 0) {
      const double gk = g[q];
      const double mk = __dadd_rn(__dmul_rn(b1, m[q]), __dmul_rn(1.0 - b1, gk));
      const double vk = __dadd_rn(__dmul_rn(b2, v[q]), __dmul_rn(1.0 - b2, __dmul_rn(gk, gk)));
      m[q] = mk;
      v[q] = vk;
      p[q] = __dsub_rn(p[q], __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mk, bc[k])),
                                       __dadd_rn(sqrt(__ddiv_rn(vk, bc[kChunk + k])), eps)));
    }
  }
}

// stopped 2 -> 1 once every block of the update kernel has run (next kernel)
__global__ void rot_seal_kernel(RotState* st) {
  if (st->stopped == 2) st->stopped = 1;
}

__global__ void rot_grad_check_kernel(const double* __restrict__ g, int64_t n6, RotState* st,
                                      int32_t* flag) {
  if (st->stopped == 1 || *flag) return;
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q < n6 && !isfinite(g[q])) raise_flag(flag, FM_ERR_NONFINITE_GRAD);
}

int check_rot_graph(const fm_rot_graph* g) {
  FM_REQUIRE(g && g->n_nodes >= 0 && g->n_edges >= 0, "bad rotation graph");
  FM_REQUIRE(g->n_edges > 0, "rotation graph has no edges");
  return FM_OK;
}

int enqueue_rot_steps(const fm_rot_graph& g, double* p6, const RotScratch& s, int steps, double lr,
                      double b1, double b2, double eps, double* history, int32_t* flag,
                      cudaStream_t st) {
  const int n = g.n_nodes;
  const int64_t n6 = (int64_t)n * 6;
  for (int k = 0; k < steps; ++k) {
    rot_R_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(p6, n, s.R, s.st, flag);
    rot_node_kernel<<<(unsigned)ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(g, p6, s.R, s.g6, s.lpart,
                                                                             s.st, flag);
    rot_loss_kernel<<<1, 256, 0, st>>>(s.lpart, n, g.n_edges, nullptr, history, s.st, flag);
    rot_grad_check_kernel<<<(unsigned)ceil_div(n6, 256), 256, 0, st>>>(s.g6, n6, s.st, flag);
    rot_adam_kernel<<<(unsigned)ceil_div(n6, 256), 256, 0, st>>>(p6, s.m, s.v, s.best, s.g6, n6, lr, b1,
                                                                b2, eps, s.bc, k, s.st, flag);
    rot_seal_kernel<<<1, 1, 0, st>>>(s.st);
    FM_LAUNCHED(rot_steps);
  }
  return FM_OK;
}

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_rot_scratch_bytes(int32_t n_nodes, int64_t n_edges) {
  (void)n_edges;
  return rot_need(n_nodes);
}

int fm_rot_loss_grad(const fm_rot_graph* g, const double* params6, double* loss_out,
                     double* grad_out, int32_t* flag, void* scratch, size_t scratch_bytes,
                     void* stream) {
  if (int rc = check_rot_graph(g)) return rc;
  FM_REQUIRE(params6 && loss_out && grad_out && flag, "null rotation loss argument");
  RotScratch s;
  FM_REQUIRE(rot_carve(g->n_nodes, scratch, scratch_bytes, s), "rotation scratch too small");
  cudaStream_t st = as_stream(stream);
  const int n = g->n_nodes;
  if (n == 0) return FM_OK;
  rot_R_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(params6, n, s.R, nullptr, flag);
  rot_node_kernel<<<(unsigned)ceil_div((int64_t)n * 32, 256), 256, 0, st>>>(*g, params6, s.R, grad_out,
                                                                           s.lpart, nullptr, flag);
  rot_loss_kernel<<<1, 256, 0, st>>>(s.lpart, n, g->n_edges, loss_out, nullptr, nullptr, flag);
  FM_LAUNCHED(rot_loss_grad);
  return FM_OK;
}

int fm_rot_refine(const fm_rot_graph* g, double* params6, int32_t max_steps, double lr,
                  double beta1, double beta2, double eps, double* history_out,
                  int32_t* steps_out, int32_t* flag, void* scratch, size_t scratch_bytes,
                  void* stream) {
  if (int rc = check_rot_graph(g)) return rc;
  FM_REQUIRE(params6 && history_out && steps_out && flag && max_steps >= 0, "bad rotation refine arguments");
  RotScratch s;
  FM_REQUIRE(rot_carve(g->n_nodes, scratch, scratch_bytes, s), "rotation scratch too small");
  cudaStream_t st = as_stream(stream);
  const int n = g->n_nodes;
  const size_t n6 = (size_t)n * 6;
  *steps_out = 0;
  if (n == 0 || max_steps == 0) return FM_OK;
  FM_CUDA(cudaMemsetAsync(s.m, 0, n6 * sizeof(double), st));
  FM_CUDA(cudaMemsetAsync(s.v, 0, n6 * sizeof(double), st));
  FM_CUDA(cudaMemcpyAsync(s.best, params6, n6 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const RotState init{INFINITY, 0, 0, 0, 0};
  FM_CUDA(cudaMemcpyAsync(s.st, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  std::vector<double> bc(2 * kChunk, 1.0);
  cudaGraphExec_t exec = nullptr;
  RotState host{};
  int done = 0;
  while (done < max_steps) {
    const int chunk = std::min(kChunk, max_steps - done);
    for (int k = 0; k < chunk; ++k) {
      const double t = (double)(done + k + 1);
      bc[k] = 1.0 - pow(beta1, t);
      bc[kChunk + k] = 1.0 - pow(beta2, t);
    }
    FM_CUDA(cudaMemcpyAsync(s.bc, bc.data(), bc.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    if (chunk == kChunk) {
      if (!exec) {
        cudaStream_t cs;
        FM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        FM_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_rot_steps(*g, params6, s, chunk, lr, beta1, beta2, eps, history_out, flag, cs);
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
      }
      FM_CUDA(cudaGraphLaunch(exec, st));
    } else if (int rc = enqueue_rot_steps(*g, params6, s, chunk, lr, beta1, beta2, eps, history_out, flag, st)) {
      if (exec) cudaGraphExecDestroy(exec);
      return rc;
    }
    done += chunk;
    FM_CUDA(cudaMemcpyAsync(&host, s.st, sizeof(host), cudaMemcpyDeviceToHost, st));
    FM_CUDA(cudaStreamSynchronize(st));
    if (host.stopped) break;
  }
  if (exec) cudaGraphExecDestroy(exec);
  *steps_out = host.steps;
  FM_CUDA(cudaMemcpyAsync(params6, s.best, n6 * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return FM_OK;
}

}  // extern "C"
