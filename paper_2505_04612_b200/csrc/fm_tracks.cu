// Track building (SURVEY 8f "next" #2): the connected components of the
// keypoint match graph that build_tracks (ref/tracks.py:38-56) finds with a
// Python union-find.  Nodes are (image, keypoint) ids, edges the
// correspondences.  Hook-and-compress on the device: every edge hooks the
// larger of its two roots under the smaller (atomicMin), then every node
// jumps to its root; repeated until no edge hooks.  Roots only ever move to
// smaller ids, so each component ends labelled by its smallest node id.
#include "fm_common.cuh"

namespace fm {
namespace {

__global__ void cc_init(int32_t n, int32_t* __restrict__ lab) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lab[i] = i;
}

__device__ __forceinline__ int32_t cc_root(const int32_t* lab, int32_t x) {
  int32_t p = __ldcg(lab + x);
  while (p != x) {
    x = p;
    p = __ldcg(lab + x);
  }
  return x;
}

__global__ void cc_hook(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                        int32_t* lab, int32_t* changed) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m) return;
  int32_t a = cc_root(lab, u[e]), b = cc_root(lab, v[e]);
  while (a != b) {
    const int32_t hi = a > b ? a : b, lo = a > b ? b : a;
    const int32_t old = atomicMin(lab + hi, lo);
    if (old == hi) {  // hi was a root and now hangs under lo
      *changed = 1;
      break;
    }
    // hi was hooked meanwhile: retry from the new roots
    a = cc_root(lab, old);
    b = cc_root(lab, lo);
  }
}

__global__ void cc_compress(int32_t n, int32_t* lab) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) lab[i] = cc_root(lab, i);
}

}  // namespace
}  // namespace fm

using namespace fm;

extern "C" {

int fm_cc_labels(int32_t n_nodes, int64_t n_edges, const int32_t* u, const int32_t* v,
                 int32_t* labels, void* stream) {
  FM_REQUIRE(n_nodes >= 0 && n_edges >= 0, "bad component sizes");
  if (n_nodes == 0) return FM_OK;
  FM_REQUIRE(labels && (n_edges == 0 || (u && v)), "null component pointer");
  cudaStream_t st = as_stream(stream);
  const unsigned nb = (unsigned)ceil_div(n_nodes, 256);
  cc_init<<<nb, 256, 0, st>>>(n_nodes, labels);
  FM_LAUNCHED(cc_init);
  if (n_edges == 0) return FM_OK;
  int32_t* flag = nullptr;
  FM_CUDA(cudaMallocAsync(&flag, sizeof(int32_t), st));
  int rc = FM_OK;
  bool converged = false;
  for (int round = 0; round < 64 && !converged; ++round) {
    int32_t h = 0;
    if (cudaMemsetAsync(flag, 0, sizeof(int32_t), st) != cudaSuccess) { rc = FM_ERR_CUDA; break; }
    cc_hook<<<(unsigned)ceil_div(n_edges, 256), 256, 0, st>>>(n_edges, u, v, labels, flag);
    cc_compress<<<nb, 256, 0, st>>>(n_nodes, labels);
    if (cudaMemcpyAsync(&h, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = FM_ERR_CUDA;
      break;
    }
    converged = !h;
  }
  cudaFreeAsync(flag, st);
  if (rc != FM_OK) return set_error(rc, "connected components: %s", cudaGetErrorString(cudaGetLastError()));
  FM_REQUIRE(converged, "connected components did not converge in 64 rounds");
  FM_LAUNCHED(cc_compress);
  return FM_OK;
}

}  // extern "C"
