// Issue-rate micro-benchmark of the point pass' per-point math, isolated from
// memory: cycles per point per SM sub-partition for (a) the fp32 moment stream
// (15 FFMA2 + 3 FADD2 + prep), (b) the same with scalar FFMA, (c) the fp64
// residual head (4 F2F + 8 DFMA + compare/L1 + weight), (d) head + fp32 moments.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/moment_bench tools/moment_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kPts = 1024;
__device__ __forceinline__ float2 f2(float s) { return make_float2(s, s); }

template <int MODE>  // 0 ffma2 moments, 1 scalar moments, 2 head only, 3 head + ffma2 moments
__global__ void k(float* out, const double* __restrict__ gin, float seed) {
  float2 M[18];
  float Ms[36];
#pragma unroll
  for (int i = 0; i < 18; ++i) M[i] = f2(0.f);
#pragma unroll
  for (int i = 0; i < 36; ++i) Ms[i] = 0.f;
  double G[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) G[i] = gin[i];
  double l1 = 0;
  float a = seed + threadIdx.x * 1e-3f, b = seed * 0.5f, c = seed * 0.25f, d = seed + 0.125f;
#pragma unroll 4
  for (int p = 0; p < kPts; ++p) {
    a = a * 0.999f + 1e-4f; b = b * 0.998f + 2e-4f; c = c * 0.997f + 3e-4f; d = d * 0.996f + 4e-4f;
    float w = 1.f;
    if (MODE >= 2) {
      const double A = a, B = b, C = c, D = d;
      const double y0 = fma(G[0], A, fma(G[1], B, G[2]));
      const double y1 = fma(G[3], A, fma(G[4], B, G[5]));
      const double y2 = fma(G[6], A, fma(G[7], B, G[8]));
      const double r = fma(C, y0, fma(D, y1, y2));
      const bool keep = fabs(r) <= 0.01;
      l1 += fabs(r);
      float rf = (float)r;
      float wr;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(wr) : "f"(fmaxf(fabsf(rf), 1e-6f)));
      w = keep ? wr : 0.f;
    }
    if (MODE == 0 || MODE == 3) {
      const float2 X1 = make_float2(a, b), X2 = make_float2(c, d);
      const float2 PQ = __fmul2_rn(f2(w), X2);
      const float2 Bp[3] = {__fmul2_rn(PQ, X2), PQ, make_float2(PQ.x * d, w)};
      const float2 AA = __fmul2_rn(f2(a), X1);
      const float Av[5] = {AA.x, AA.y, a, b * b, b};
#pragma unroll
      for (int j = 0; j < 5; ++j)
#pragma unroll
        for (int q = 0; q < 3; ++q) M[j * 3 + q] = __ffma2_rn(f2(Av[j]), Bp[q], M[j * 3 + q]);
#pragma unroll
      for (int q = 0; q < 3; ++q) M[15 + q] = __fadd2_rn(Bp[q], M[15 + q]);
    }
    if (MODE == 1) {
      const float p_ = w * c, q_ = w * d;
      const float Bv[6] = {p_ * c, p_ * d, p_, q_ * d, q_, w};
      const float Av[6] = {a * a, a * b, a, b * b, b, 1.f};
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j) Ms[i * 6 + j] = fmaf(Bv[i], Av[j], Ms[i * 6 + j]);
    }
  }
  float s = (float)l1;
#pragma unroll
  for (int i = 0; i < 18; ++i) s += M[i].x + M[i].y;
#pragma unroll
  for (int i = 0; i < 36; ++i) s += Ms[i];
  if (s == 1.2345f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* buf;
  double* g;
  cudaMalloc(&buf, 64);
  cudaMalloc(&g, 9 * sizeof(double));
  double hg[9] = {0.1, -0.2, 0.3, 0.05, 0.7, -0.1, 0.2, 0.01, -0.6};
  cudaMemcpy(g, hg, sizeof(hg), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"ffma2 moments", "scalar moments", "fp64 head", "head+ffma2 mom"};
  void (*ks[4])(float*, const double*, float) = {k<0>, k<1>, k<2>, k<3>};
  for (int m = 0; m < 4; ++m) {
    for (int warps : {8, 12, 16, 24}) {
      const int threads = 128, blocks = sms * warps / 4;
      ks[m]<<<blocks, threads>>>(buf, g, 1.5f);
      cudaEventRecord(e0);
      ks[m]<<<blocks, threads>>>(buf, g, 1.5f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double pts_per_smsp = (double)blocks * threads * kPts / (sms * 4);
      const double cyc = ms * 1e-3 * clk * 1e3;
      printf("%-16s warps/SM %2d: %.3f ms, %.2f SMSP-cycles per 32 points (warp-point)\n", names[m], warps,
             ms, cyc / (pts_per_smsp / 32));
    }
  }
  cudaFuncAttributes fa;
  for (int m = 0; m < 4; ++m) { cudaFuncGetAttributes(&fa, ks[m]); printf("%s regs %d\n", names[m], fa.numRegs); }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
