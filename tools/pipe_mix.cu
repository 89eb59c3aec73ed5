// Which pipes does the point pass's per-point mix contend on?  Each kernel runs
// NF2F cvt.f64.f32, NRCP rcp.approx, NDFMA fp64 FMA, NFF2 FFMA2 (packed fp32),
// NDMMA mma.sync m8n8k4 f64 and NALU integer LOP3/IADD per iteration on
// independent chains; prints SMSP-cycles per warp-iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pm tools/pipe_mix.cu && /tmp/pm
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIt = 1024;

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  return __ffma2_rn(a, b, c);
}

template <int NF2F, int NRCP, int NDFMA, int NFF2, int NDMMA, int NALU, int NFF = 0, int NIMAD = 0>
__global__ void k(float* out, float seed) {
  float y[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) y[i] = seed * i + threadIdx.x;
  const float ym = seed * 0.5f + threadIdx.x * 1e-7f;
  float f[8];
  double dd[8];
  float r[8];
  float2 x[16];
  double c[8][2];
  unsigned u[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[i] = seed + i + threadIdx.x; dd[i] = f[i]; r[i] = f[i] + 1;
    c[i][0] = c[i][1] = f[i]; u[i] = threadIdx.x * 7 + i;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = make_float2(seed * i, seed + i);
  const float2 m = make_float2(1.0000001f, 0.9999999f), a2 = make_float2(1e-9f, 2e-9f);
  for (int it = 0; it < kIt; ++it) {
#pragma unroll
    for (int i = 0; i < NF2F; ++i) {
      double v;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(v) : "f"(f[i % 8]));
      f[i % 8] = __int_as_float(__double2hiint(v) ^ 0x1);
    }
#pragma unroll
    for (int i = 0; i < NRCP; ++i) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(r[i % 8]));
#pragma unroll
    for (int i = 0; i < NDFMA; ++i) dd[i % 8] = fma(dd[i % 8], 1.0000001, 1e-9);
#pragma unroll
    for (int i = 0; i < NFF2; ++i) x[i % 16] = ffma2(x[i % 16], m, a2);
#pragma unroll
    for (int i = 0; i < NDMMA; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i % 8][0]), "+d"(c[i % 8][1])
                   : "d"(1.0000001), "d"(dd[0]));
#pragma unroll
    for (int i = 0; i < NFF; ++i) y[i % 16] = fmaf(y[i % 16], ym, 1e-9f);
#pragma unroll
    for (int i = 0; i < NIMAD; ++i) u[i % 8] = u[i % 8] * 0x9e3779b1u + it;
#pragma unroll
    for (int i = 0; i < NALU; ++i) asm volatile("lop3.b32 %0, %0, %1, 0x5a5a5a5a, 0x96;" : "+r"(u[i % 8]) : "r"(it));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i] + (float)dd[i] + r[i] + (float)c[i][0] + (float)c[i][1] + u[i];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i].x + x[i].y;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += y[i];
  if (s == 1.2345f) out[0] = s;
}

template <int A, int B, int C, int D, int E, int F, int G = 0, int H = 0>
void run(const char* name, int sms, int clk, float* buf) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 512, blocks = sms * 2;  // 32 warps / SM
  k<A, B, C, D, E, F, G, H><<<blocks, threads>>>(buf, 1.5f);
  cudaEventRecord(e0);
  k<A, B, C, D, E, F, G, H><<<blocks, threads>>>(buf, 1.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warp_its_per_smsp = (double)blocks * threads / 32 * kIt / (sms * 4);
  printf("%-34s %7.2f SMSP-cycles per warp-iteration\n", name, ms * 1e-3 * clk * 1e3 / warp_its_per_smsp);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* buf;
  cudaMalloc(&buf, 64);
  run<8, 0, 0, 0, 0, 0>("8 F2F", sms, clk, buf);
  run<0, 8, 0, 0, 0, 0>("8 RCP", sms, clk, buf);
  run<0, 0, 8, 0, 0, 0>("8 DFMA", sms, clk, buf);
  run<0, 0, 0, 16, 0, 0>("16 FFMA2", sms, clk, buf);
  run<0, 0, 0, 0, 8, 0>("8 DMMA", sms, clk, buf);
  run<0, 0, 0, 0, 0, 16>("16 LOP3", sms, clk, buf);
  run<0, 0, 8, 16, 0, 0>("8 DFMA + 16 FFMA2", sms, clk, buf);
  run<8, 0, 0, 16, 0, 0>("8 F2F + 16 FFMA2", sms, clk, buf);
  run<0, 0, 0, 16, 8, 0>("8 DMMA + 16 FFMA2", sms, clk, buf);
  run<0, 0, 8, 0, 8, 0>("8 DMMA + 8 DFMA", sms, clk, buf);
  run<0, 0, 0, 16, 0, 16>("16 LOP3 + 16 FFMA2", sms, clk, buf);
  run<8, 0, 8, 0, 0, 0>("8 F2F + 8 DFMA", sms, clk, buf);
  // the pass's per-point mix (x4 points): 5 F2F, 1 RCP, 8 DFMA, 26 FFMA2-class, ~25 ALU
  run<20, 4, 32, 104, 0, 0>("pass mix x4 without ALU", sms, clk, buf);
  run<20, 4, 32, 104, 0, 100>("pass mix x4 with 100 ALU", sms, clk, buf);
  run<20, 4, 0, 104, 8, 0>("pass mix x4, DFMA -> 8 DMMA", sms, clk, buf);
  run<0, 0, 0, 0, 0, 0, 32, 0>("32 FFMA", sms, clk, buf);
  run<0, 0, 0, 0, 0, 0, 32, 0>("32 FFMA (again)", sms, clk, buf);
  run<0, 0, 0, 16, 0, 0, 0, 0>("16 FFMA2 (again)", sms, clk, buf);
  run<0, 0, 0, 0, 0, 16, 32, 0>("32 FFMA + 16 LOP3", sms, clk, buf);
  run<0, 0, 0, 0, 0, 0, 0, 16>("16 IMAD", sms, clk, buf);
  run<0, 0, 0, 16, 0, 0, 0, 16>("16 FFMA2 + 16 IMAD", sms, clk, buf);
  run<0, 0, 0, 0, 0, 0, 32, 16>("32 FFMA + 16 IMAD", sms, clk, buf);
  run<0, 0, 8, 0, 0, 0, 32, 0>("8 DFMA + 32 FFMA", sms, clk, buf);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
