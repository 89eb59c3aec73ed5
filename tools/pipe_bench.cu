// Pipe-throughput micro-benchmark (per SM per clock) for the instructions the
// point pass is made of: DFMA, F2F.F64.F32, DMUL, FFMA2, MUFU.RCP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pb tools/pipe_bench.cu && /tmp/pb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

__global__ void dfma_k(double* out, double a, double b) {
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

__global__ void f2f_k(double* out, float a) {
  float f[16];
  double acc[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 16; ++k) f[k] = threadIdx.x * 0.001f + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      f[k] = f[k] * a;  // dependency to keep the conversion live
      acc[k & 3] += (double)f[k];
    }
  }
  if (acc[0] + acc[1] + acc[2] + acc[3] == 1.2345) out[0] = acc[0];
}

__global__ void ffma2_k(float2* out, float2 a, float2 b) {
  float2 x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = make_float2(threadIdx.x + k, k);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = __ffma2_rn(x[k], a, b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k].x + x[k].y;
  if (s == 1.2345f) out[0] = x[0];
}

__global__ void ffma_k(float* out, float a, float b) {
  float x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 1.2345f) out[0] = s;
}

// 8 FFMA2 chains + 8 scalar FFMA chains: does scalar FFMA use a pipe FFMA2 leaves free?
__global__ void mix_k(float* out, float2 a, float2 b) {
  float2 x[8];
  float y[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { x[k] = make_float2(threadIdx.x + k, k); y[k] = threadIdx.x - k; }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { x[k] = __ffma2_rn(x[k], a, b); y[k] = fmaf(y[k], a.x, b.x); }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y + y[k];
  if (s == 1.2345f) out[0] = s;
}

// fp32 -> fp64 conversions with no other work (XU rate)
__global__ void cvt_k(double* out, float a) {
  double x[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) x[k] = 0;
  float f = a + threadIdx.x;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { x[k] = (double)f; f = __int_as_float(__float_as_int(f) ^ (k + 1)); }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += x[k];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void* buf;
  cudaMalloc(&buf, 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch, double ops_per_thread_iter, int blocks, int threads) {
    launch(blocks, threads);
    cudaEventRecord(e0);
    launch(blocks, threads);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = ops_per_thread_iter * kIters * (double)blocks * threads;
    double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
    printf("%-10s %8.3f ms  %.3e ops/s  %.1f lane-ops/clk/SM (at max clock %d MHz)\n", name, ms,
           ops / (ms * 1e-3), per_clk_sm, clk / 1000);
  };
  for (int threads : {256, 512, 1024}) {
    printf("threads/block %d, blocks %d\n", threads, sms * 4);
    run("DFMA", [&](int b, int t) { dfma_k<<<b, t>>>((double*)buf, 1.0000001, 1e-9); }, 16, sms * 4, threads);
    run("F2F+DADD", [&](int b, int t) { f2f_k<<<b, t>>>((double*)buf, 1.0000001f); }, 16, sms * 4, threads);
    run("FFMA2(x2)", [&](int b, int t) { ffma2_k<<<b, t>>>((float2*)buf, make_float2(1.0000001f, 1.0f), make_float2(1e-9f, 0.f)); }, 32, sms * 4, threads);
    run("FFMA", [&](int b, int t) { ffma_k<<<b, t>>>((float*)buf, 1.0000001f, 1e-9f); }, 16, sms * 4, threads);
    run("FFMA2+FFMA", [&](int b, int t) { mix_k<<<b, t>>>((float*)buf, make_float2(1.0000001f, 1.0f), make_float2(1e-9f, 0.f)); }, 24, sms * 4, threads);
    run("F2F only", [&](int b, int t) { cvt_k<<<b, t>>>((double*)buf, 1.0000001f); }, 16, sms * 4, threads);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
