// Does the fp64 tensor-core MMA (mma.sync m8n8k4 f64, SASS DMMA) run on a
// pipe separate from the fp64 vector FMA (DFMA)?  Measures DMMA alone, DFMA
// alone and both interleaved, in FMAs per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/db tools/dmma_bench.cu && /tmp/db
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NMMA, int NFMA>
__global__ void mix_k(double* out, double a, double b) {
  double c[8][2];
  double x[16];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x + k;
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 0.5 + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < NMMA; ++k) dmma(c[k], a + k, b);
#pragma unroll
    for (int k = 0; k < NFMA; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* buf;
  cudaMalloc(&buf, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(double*, double, double), int nmma, int nfma) {
    const int blocks = sms * 4, threads = 256;
    k<<<blocks, threads>>>(buf, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    k<<<blocks, threads>>>(buf, 1.0000001, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warps = (double)blocks * threads / 32;
    const double mma_fma = warps * kIters * nmma * 256.0;   // m8n8k4 = 256 FMAs
    const double vec_fma = warps * 32 * kIters * (double)nfma;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-18s %8.3f ms  DMMA %.1f  DFMA %.1f  total %.1f FMA/clk/SM\n", name, ms,
           mma_fma / cyc / sms, vec_fma / cyc / sms, (mma_fma + vec_fma) / cyc / sms);
  };
  run("DMMA x8", mix_k<8, 0>, 8, 0);
  run("DFMA x16", mix_k<0, 16>, 0, 16);
  run("DMMA x8 + DFMA x16", mix_k<8, 16>, 8, 16);
  run("DMMA x4 + DFMA x16", mix_k<4, 16>, 4, 16);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
