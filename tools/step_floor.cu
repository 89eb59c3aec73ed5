// Launch/ramp floor of the two-kernel Adam step: trivial kernels with the
// step's grid shapes (pair_grad 391 x 64, image_reduce 251 x 64 at C2),
// 100 steps captured in a CUDA graph, replayed; time per step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ka(const double* in, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i] * 1.0000001 + 1e-9;
}
__global__ void kb(const double* in, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[(i * 7) % n] + 1.0;
}
int main() {
  const int P = 25000, N = 16000;
  double *a, *b;
  cudaMalloc(&a, P * 8 * 24);
  cudaMalloc(&b, P * 8 * 24);
  cudaMemset(a, 0, P * 8 * 24);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int variant = 0; variant < 3; ++variant) {
    cudaGraph_t g;
    cudaGraphExec_t e;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < 100; ++k) {
      if (variant != 2) ka<<<(P + 63) / 64, 64, 0, s>>>(a, b, P);
      if (variant != 1) kb<<<(N + 63) / 64, 64, 0, s>>>(b, a, N);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&e, g, 0);
    cudaGraphLaunch(e, s);
    cudaStreamSynchronize(s);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventRecord(t0, s);
    for (int r = 0; r < 9; ++r) cudaGraphLaunch(e, s);
    cudaEventRecord(t1, s);
    cudaEventSynchronize(t1);
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    const char* name[] = {"both kernels", "pair-shaped only", "image-shaped only"};
    printf("%s: %.2f us per step\n", name[variant], ms * 1e3 / 900);
  }
  return 0;
}
