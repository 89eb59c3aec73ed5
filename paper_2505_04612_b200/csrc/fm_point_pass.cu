// Fused point-pair pass of the epipolar adjustment -- the HBM-bound hot kernel.
//
// One sweep over the structure-of-arrays point store replaces, for every
// active point pair m of image pair n,
//   current_residuals     r_m = t_m . ghat_n        (ref/epipolar.py:251-255)
//   pruning               active &= |r_m| <= th     (ref/epipolar.py:280-288)
//   epipolar_loss("l1")   sum |r_m|                 (ref/epipolar.py:156-160)
//   precompute_weights    W_n = sum w_m t_m t_m^T   (ref/epipolar.py:46-59)
// with t_m = flatten(x2 x1^T) never materialised.  W_n has Kronecker structure
// (t = x2 (x) x1), so it is carried as 36 fourth-order moments
//   mom[sym(p,q)][sym(r,s)] = sum w x2_p x2_q x1_r x1_s,
// plus the linearisation terms of the shifted quadratic model
//   vgrad = sum w r0 t  (= W ghat0),  s0 = sum w r0^2  (= ghat0^T W ghat0),
// which keep the per-step loss/gradient accurate with fp32 moments even
// though W is ill-conditioned ("shifted quadratic model").
//
// Execution (hot kernel, z == 1): one warp per work item (a <= chunk-slot
// slice of one image pair; pairs start 4-aligned so each lane moves whole
// 32-byte (x, y) groups with 128-bit non-allocating loads, software-pipelined
// one iteration ahead).  Residual, prune decision, s0 and L1 are fp64; the 45
// moment / gradient accumulators are fp32 and use Blackwell's packed FFMA2
// (fma.rn.f32x2: two FMAs per issue slot).  Warp totals come from a
// fixed-order transpose reduction -- no floating-point atomics, so results are
// bitwise reproducible run to run.
#include <cmath>
#include <cstdlib>

#include "fm_common.cuh"

namespace fm {

namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kNumRed = 46;  // 36 moments + 9 vgrad + post-prune count

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

__device__ __forceinline__ float2 f2(float s) { return make_float2(s, s); }

// 64-value variant for the generic kernel: lane l ends with values 2l, 2l+1.
template <typename T>
__device__ __forceinline__ void warp_transpose_reduce64(T (&v)[64], int lane) {
#pragma unroll
  for (int level = 0; level < 5; ++level) {
    const int off = 16 >> level;
    const int half = 32 >> level;
    const bool upper = (lane & off) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const T send = upper ? v[i] : v[i + half];
      const T keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

struct PartialBufs {
  void* red;   // [kNumRed][n_items] of the accumulator type
  double* s0;  // [n_items]
  double* l1;  // [n_items]
};

// Hot-kernel accumulator order.  x2 products (rows) and x1 products (cols)
// are both kept in the order {00, 01, 02, 12, 11, 22} so that pairs
// (x^2, xy) = x*(x, y), (x, y) and (y^2, 1) are natural float2 registers.
__device__ __forceinline__ int hot_perm(int k) { return k == 3 ? 4 : (k == 4 ? 3 : k); }

// Canonical output index of hot accumulator slot v (0..45), or -1.
// 0..35 moments (row-major 6x6 in hot order), 36..44 vgrad pairs, 45 count.
__device__ __forceinline__ int hot_out_index(int v) {
  if (v < 36) return hot_perm(v / 6) * 6 + hot_perm(v % 6);
  switch (v) {  // V0=(v00,v01) V1=(v10,v11) V2=(v20,v21) V3=(v02,v12) v22
    case 36: return 36 + 0;
    case 37: return 36 + 1;
    case 38: return 36 + 3;
    case 39: return 36 + 4;
    case 40: return 36 + 6;
    case 41: return 36 + 7;
    case 42: return 36 + 2;
    case 43: return 36 + 5;
    case 44: return 36 + 8;
    case 45: return 45;
    default: return -1;
  }
}

__device__ __forceinline__ void store_red(const fm_pass_out& out, const PartialBufs& part, bool single,
                                          int64_t P, int64_t NI, int n, int64_t item, int k, float val,
                                          bool lin) {
  if (!single) {
    static_cast<float*>(part.red)[k * NI + item] = val;
    return;
  }
  if (k < 36) {
    out.mom32[k * P + n] = val;
  } else if (k < 45) {
    if (lin) out.vgrad[(k - 36) * P + n] = val;
  } else if (out.n_active) {
    out.n_active[n] = (int32_t)val;
  }
}

// ------------------------------------------------------------------ hot kernel
// z == 1.  A warp works on 32/L consecutive work items at once: L lanes per
// item (an item is a <= chunk-slot slice of one image pair).  Each lane owns
// every L-th 4-slot group of its item and streams it through a private
// per-lane ring of kRing shared-memory stages with cp.async (LDGSTS, 16-byte
// L2-only copies, one commit group per iteration), so kRing x 64 B per lane
// are in flight without holding registers.  Per-item totals need only
// log2(L) butterfly levels across the item's lanes (fixed order -> bitwise
// reproducible), instead of a 32-lane reduction per item.
//
// MOM64 = true (default, exact): the 36 Kronecker moments accumulate in fp64,
// so W matches the reference's fp64 W to rounding -- the IRLS quadratic form
// is ill-conditioned and fp32 moments visibly move the optimum.
// MOM64 = false (opt-in fast mode): fp32 moments with packed FFMA2 plus the
// shifted-model linearisation terms vgrad / s0.
#ifndef FM_HOT_RING
#define FM_HOT_RING 5
#endif
constexpr int kRing = FM_HOT_RING;  // stages per lane
constexpr int kGrpWarps = 4;    // warps per block

__device__ __forceinline__ float and_mask(float x, unsigned m) {
  unsigned r;
  asm("and.b32 %0, %1, %2;" : "=r"(r) : "r"(__float_as_uint(x)), "r"(m));
  return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct ItemDesc {
  int64_t lo;   // first slot
  int len;      // points in the item
  int n;        // image pair
  bool single;  // the pair is one work item
};

// Descriptor {lo (2 x int32), len, n | single << 31} -> ItemDesc.
__device__ __forceinline__ ItemDesc decode_item(int4 q) {
  ItemDesc d;
  d.lo = (int64_t)(uint32_t)q.x | ((int64_t)q.y << 32);
  d.len = q.z;
  d.n = q.w & 0x7fffffff;
  d.single = (q.w >> 31) & 1;
  return d;
}

__global__ void describe_items_kernel(const fm_point_store s, int32_t* __restrict__ desc) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= s.n_items) return;
  const int n = s.item_pair[k];
  const int first = s.pair_item_off[n];
  const int c = (int)(k - first);
  const int64_t lo = s.pair_off[n] + (int64_t)c * s.chunk;
  const int64_t rem = (int64_t)s.pair_len[n] - (int64_t)c * s.chunk;
  const int len = (int)(rem < s.chunk ? rem : s.chunk);
  const bool single = (s.pair_item_off[n + 1] - first) == 1;
  int4 q;
  q.x = (int)(uint32_t)(lo & 0xffffffffll);
  q.y = (int)(lo >> 32);
  q.z = len;
  q.w = n | (single ? (int)0x80000000 : 0);
  reinterpret_cast<int4*>(desc)[k] = q;
}

// What the moment stream needs of one point, produced by the residual head
// one iteration earlier (software pipelining: the latency-bound head of
// iteration it+1 -- shared-memory loads, conversions, the fp64 residual
// chain, the reciprocal -- overlaps the independent DFMA stream of it).
struct PtCarry {
  float2 X1, X2;
  float w;   // IRLS weight, +0 for dropped / pruned / invalid slots
  float wr;  // w * r (fp32 shifted model only)
};

template <bool kPrune, bool kL1, bool kMom, bool MOM64>
struct HotAcc {
  double M64[MOM64 ? 36 : 1];
  float2 M2[MOM64 ? 1 : 18];
  float2 V0, V1, V2, V3;
  float v22, s0f;
  double l1;
  int cnt;

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < (MOM64 ? 36 : 1); ++k) M64[k] = 0.0;
#pragma unroll
    for (int k = 0; k < (MOM64 ? 1 : 18); ++k) M2[k] = f2(0.f);
    V0 = V1 = V2 = V3 = f2(0.f);
    v22 = s0f = 0.f;
    l1 = 0.0;
    cnt = 0;
  }

  // Residual head of one point pair: prune decision, count, L1, IRLS weight.
  // Returns the post-prune keep flag.  Branch-free: the residual and weight
  // are computed for every slot and masked afterwards, so the compiler can
  // interleave the independent points of an iteration.
  __device__ __forceinline__ bool head(const double (&G)[9], float2 X1, float2 X2, bool act,
                                       double thr, PtCarry& C) {
    // residual r = x2^T Ghat x1 in fp64 (ref/epipolar.py:255)
    const double a = X1.x, bb = X1.y, c = X2.x, dd = X2.y;
    const double y0 = fma(G[0], a, fma(G[1], bb, G[2]));
    const double y1 = fma(G[3], a, fma(G[4], bb, G[5]));
    const double y2 = fma(G[6], a, fma(G[7], bb, G[8]));
    const double r = fma(c, y0, fma(dd, y1, y2));
    const double ar = fabs(r);
    const bool keep = kPrune ? (act & (ar <= thr)) : act;
    cnt += keep;
    if (kL1) l1 += act ? ar : 0.0;
    C.X1 = X1;
    C.X2 = X2;
    if (kMom) {
      // IRLS weight 1/max(|r|, 1e-6) (ref/epipolar.py:58) from the rounded
      // residual: a per-point relative error of the weight keeps every term
      // rank-1 exact.  Coordinates of every slot are finite (the store
      // builders zero and deactivate non-finite points), so a zero weight
      // removes a dropped point exactly without selecting its coordinates.
      const float rf = (float)r;
      const float arf = fabsf(rf);
      const float wraw = rcp_approx(fmaxf(arf, 1e-6f));
      // opaque AND (not a select) so the compiler cannot sink the reciprocal
      // into a per-point branch and serialise the iteration's points
      C.w = and_mask(wraw, keep ? 0xffffffffu : 0u);
      if (!MOM64) {
        // w r0 = sign(r) and w r0^2 = |r| unless clamped (|r| < 1e-6)
        const bool big = arf >= 1e-6f;
        C.wr = keep ? (big ? copysignf(1.f, rf) : rf * 1e6f) : 0.f;
        s0f += keep ? (big ? arf : rf * rf * 1e6f) : 0.f;
      }
    }
    return keep;
  }

  // Moment stream of one point: W += w t t^T as the 36 Kronecker moments
  // (plus the shifted-model vgrad terms in fp32 mode).
  __device__ __forceinline__ void stream(const PtCarry& C) {
    if (!kMom) return;
    const float2 Y1 = C.X1, Y2 = C.X2;
    if (MOM64) {
      const double w = C.w;
      const double ka = Y1.x, kb = Y1.y, kc = Y2.x, kd = Y2.y;
      const double A[6] = {ka * ka, ka * kb, ka, kb * kb, kb, 1.0};
      const double wc = w * kc, wd = w * kd;
      const double B[6] = {wc * kc, wc * kd, wc, wd * kd, wd, w};
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = 0; j < 6; ++j)
          M64[MOM64 ? i * 6 + j : 0] = fma(B[i], A[j], M64[MOM64 ? i * 6 + j : 0]);
    } else {
      const float wf = C.w, wr = C.wr;
      const float2 wX2 = __fmul2_rn(f2(wf), Y2);
      const float B[6] = {wX2.x * Y2.x, wX2.x * Y2.y, wX2.x, wX2.y * Y2.y, wX2.y, wf};
      const float2 A0 = __fmul2_rn(f2(Y1.x), Y1);
      const float2 A2 = make_float2(Y1.y * Y1.y, 1.f);
      const float Brow[6] = {B[0], B[1], B[2], B[4], B[3], B[5]};
#pragma unroll
      for (int p = 0; p < 6; ++p) {
        M2[MOM64 ? 0 : p * 3 + 0] = __ffma2_rn(f2(Brow[p]), A0, M2[MOM64 ? 0 : p * 3 + 0]);
        M2[MOM64 ? 0 : p * 3 + 1] = __ffma2_rn(f2(Brow[p]), Y1, M2[MOM64 ? 0 : p * 3 + 1]);
        M2[MOM64 ? 0 : p * 3 + 2] = __ffma2_rn(f2(Brow[p]), A2, M2[MOM64 ? 0 : p * 3 + 2]);
      }
      const float2 wrX2 = __fmul2_rn(f2(wr), Y2);
      V0 = __ffma2_rn(f2(wrX2.x), Y1, V0);
      V1 = __ffma2_rn(f2(wrX2.y), Y1, V1);
      V2 = __ffma2_rn(f2(wr), Y1, V2);
      V3 = __fadd2_rn(wrX2, V3);
      v22 += wr;
    }
  }
};

// Per-lane ring: stage d holds the lane's NPT slots of x1 and x2 (NPT/2
// 16-byte chunks each) and the mask words, laid out chunk-major so that a
// warp's LDS.128 of one chunk touches 32 consecutive 16-byte words (no bank
// conflicts).
#ifndef FM_HOT_NPT
#define FM_HOT_NPT 4
#endif
#ifndef FM_HOT_GSM
#define FM_HOT_GSM 0
#endif
#ifndef FM_HOT_NOLOAD
#define FM_HOT_NOLOAD 0  // tuning experiment only: skip the global loads
#endif
#ifndef FM_HOT_MINB
#define FM_HOT_MINB 3
#endif
constexpr int kNpt = FM_HOT_NPT;   // points per lane per iteration (2 or 4)
constexpr bool kGsm = FM_HOT_GSM;  // ghat of the warp's items in shared memory
struct LaneRing {
  float4 c[kRing][kNpt][32];     // [stage][chunk: x1 (NPT/2), x2 (NPT/2)][lane]
  uint32_t m[kRing][kNpt / 2][32];  // mask word of each slot pair
  double G[kGsm ? 32 : 1][9];     // ghat of the warp's items (kGsm)
};

template <int L>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int off = 1; off < L; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}
template <int L>
__device__ __forceinline__ float group_sumf(float x) {
#pragma unroll
  for (int off = 1; off < L; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

template <unsigned MODE, bool MOM64, int L>
__global__ void __launch_bounds__(kGrpWarps * 32, FM_HOT_MINB)
point_pass_hot(const fm_point_store s, const double* __restrict__ ghat, const double thr,
               const int32_t* __restrict__ prev_active, const fm_pass_out out,
               const PartialBufs part) {
  constexpr bool kPrune = MODE & FM_PASS_PRUNE;
  constexpr bool kL1 = MODE & FM_PASS_L1;
  constexpr bool kMom = (MODE & FM_PASS_MOMENTS) && (MODE & FM_PASS_IRLS);
  constexpr bool kLin = kMom && !MOM64;
  constexpr bool kSkip = MODE & FM_PASS_SKIP_DROPPED;
  constexpr int IPW = 32 / L;        // items per warp
  constexpr int kPairs = kNpt / 2;   // slot pairs (16-byte chunks per column) per lane
  constexpr int kBlk = kNpt * L;     // slots per group iteration

  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  LaneRing& ring = reinterpret_cast<LaneRing*>(smem_raw)[wib];
  const int64_t P = s.n_pairs;
  const int64_t NI = s.n_items;
  const int g = lane % L;  // lane within the item group
  const int q = lane / L;  // item within the warp
  const int64_t item = ((int64_t)blockIdx.x * kGrpWarps + wib) * IPW + q;
  const bool has_item = item < NI;

  ItemDesc d{0, 0, 0, true};
  if (has_item) d = decode_item(__ldg(reinterpret_cast<const int4*>(s.item_desc) + item));
  const bool skip = has_item && kSkip && prev_active[d.n] == 0;
  double G[kGsm ? 1 : 9];
  if (kGsm) {
    for (int k = g; k < 9; k += L) ring.G[q][k] = (has_item && !skip) ? ghat[k * P + d.n] : 0.0;
  } else {
#pragma unroll
    for (int k = 0; k < (kGsm ? 1 : 9); ++k) G[k] = (has_item && !skip) ? ghat[k * P + d.n] : 0.0;
  }
  // iterations of this group: kBlk-slot blocks of the item (same for its lanes)
  const int len = (has_item && !skip) ? d.len : 0;
  const int nit = (len + kBlk - 1) / kBlk;
  const int warp_it = __reduce_max_sync(0xffffffffu, nit);
  const int lo_lo = (int)(d.lo & 31);  // slot offsets below are item-relative int32
  const float4* x1b = reinterpret_cast<const float4*>(s.x1 + 2 * d.lo) + g;
  const float4* x2b = reinterpret_cast<const float4*>(s.x2 + 2 * d.lo) + g;
  const uint32_t* mwb = reinterpret_cast<const uint32_t*>(s.active) + (d.lo >> 5);
  uint32_t* mwb_w = reinterpret_cast<uint32_t*>(s.active) + (d.lo >> 5);

  // Iteration `it` of a group covers the kBlk-slot block at d.lo + kBlk*it;
  // lane g copies 16-byte chunks g + L*j (j < NPT/2) of each column, so each
  // copy instruction of the group reads whole 32-byte sectors; the lane owns
  // slot pairs {2(g + L j), 2(g + L j) + 1}.  Every lane reads back only the
  // ring slots it copied itself, so cp.async.wait_group suffices (no warp
  // barrier).  Shared addresses are 32-bit and hoisted; the ring stage is a
  // running index.
  constexpr uint32_t kChunkB = 32 * 16;              // one chunk row of the warp
  constexpr uint32_t kStageC = kNpt * kChunkB;       // coordinate bytes per stage
  constexpr uint32_t kStageM = kPairs * 32 * 4;      // mask bytes per stage
  const uint32_t ring_c = smem_u32(&ring.c[0][0][lane]);
  const uint32_t ring_m = smem_u32(&ring.m[0][0][lane]);
  auto issue = [&](int it, uint32_t st) {  // st = stage index
    if (FM_HOT_NOLOAD == 0 && it < nit) {
      const float4* p1 = x1b + (kBlk / 2) * it;
      const float4* p2 = x2b + (kBlk / 2) * it;
#pragma unroll
      for (int j = 0; j < kPairs; ++j) {
        // chunks at or past the item end are not fetched (they may lie past
        // the allocation); their stale stage bytes are finite and masked
        const int off = kBlk * it + 2 * (g + L * j);
        if (off < len) {
          cp_async16(ring_c + st * kStageC + j * kChunkB, p1 + L * j);
          cp_async16(ring_c + st * kStageC + (kPairs + j) * kChunkB, p2 + L * j);
          cp_async4(ring_m + st * kStageM + j * 128, mwb + ((lo_lo + off) >> 5));
        }
      }
    }
    cp_async_commit();
  };
  {  // stale stage bytes must be finite: zero this lane's ring slots once
#pragma unroll
    for (int st = 0; st < kRing; ++st)
#pragma unroll
      for (int c = 0; c < kNpt; ++c) ring.c[st][c][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < kRing - 1; ++it) issue(it, it);

  HotAcc<kPrune, kL1, kMom, MOM64> acc;
  acc.zero();
  uint32_t st_issue = kRing - 1, st_read = 0;
#pragma unroll 1
  for (int it = 0; it < warp_it; ++it) {
    issue(it + kRing - 1, st_issue);
    st_issue = st_issue + 1 == kRing ? 0 : st_issue + 1;
    cp_async_wait<kRing - 1>();  // this lane's copies of iteration `it` have landed
    // Past the item end (it >= nit, or a lane group without an item) every
    // slot-valid bit is 0: nothing counts, nothing is pruned, weights are +0.
    double Gl[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) Gl[k] = kGsm ? ring.G[q][k] : G[kGsm ? 0 : k];
    PtCarry C[kNpt];
#pragma unroll
    for (int j = 0; j < kPairs; ++j) {
      const int off = kBlk * it + 2 * (g + L * j);
      const int sh = (lo_lo + off) & 31;
      const int la = len - off;
      const unsigned va = la >= 2 ? 3u : (la > 0 ? 1u : 0u);
      const unsigned bits = FM_HOT_NOLOAD ? va : (lds32(ring_m + st_read * kStageM + j * 128) >> sh) & va;
      const float4 a = lds128(ring_c + st_read * kStageC + j * kChunkB);
      const float4 b = lds128(ring_c + st_read * kStageC + (kPairs + j) * kChunkB);
      unsigned keep_bits = (unsigned)acc.head(Gl, make_float2(a.x, a.y), make_float2(b.x, b.y),
                                              bits & 1u, thr, C[2 * j]);
      keep_bits |= (unsigned)acc.head(Gl, make_float2(a.z, a.w), make_float2(b.z, b.w),
                                      (bits >> 1) & 1u, thr, C[2 * j + 1]) << 1;
      if (kPrune) {
        const unsigned cleared = bits & ~keep_bits;
        if (cleared) atomicAnd(mwb_w + ((lo_lo + off) >> 5), ~(cleared << sh));
      }
    }
    st_read = st_read + 1 == kRing ? 0 : st_read + 1;
#pragma unroll
    for (int k = 0; k < kNpt; ++k) acc.stream(C[k]);
  }
  cp_async_wait<0>();

  // ------------------------------------------------------------------ reduce
  // log2(L) butterfly levels within the item's lanes; lane g then writes
  // outputs k = g, g + L, ... (consecutive items -> coalesced SoA stores)
  const bool single = d.single;
  if (kMom && MOM64) {
    double v[38];
#pragma unroll
    for (int k = 0; k < 36; ++k) v[k] = group_sum<L>(acc.M64[MOM64 ? k : 0]);
    v[36] = group_sum<L>((double)acc.cnt);
    v[37] = group_sum<L>(acc.l1);
    if (has_item) {
#pragma unroll
      for (int k = 0; k < 38; ++k) {
        if (k % L != g) continue;
        if (!single) {
          if (k < 36) static_cast<double*>(part.red)[k * NI + item] = v[k];
          else if (k == 36) static_cast<double*>(part.red)[45 * NI + item] = v[k];
          else part.l1[item] = v[k];
        } else if (k < 36) {
          out.mom64[k * P + d.n] = v[k];
        } else if (k == 36) {
          if (out.n_active) out.n_active[d.n] = (int32_t)v[k];
        } else if (kL1 && out.l1) {
          out.l1[d.n] = v[k];
        }
      }
    }
  } else if (kMom) {
    float v[47];
#pragma unroll
    for (int k = 0; k < 18; ++k) {
      v[2 * k] = group_sumf<L>(acc.M2[MOM64 ? 0 : k].x);
      v[2 * k + 1] = group_sumf<L>(acc.M2[MOM64 ? 0 : k].y);
    }
    const float vv[11] = {acc.V0.x, acc.V0.y, acc.V1.x, acc.V1.y, acc.V2.x, acc.V2.y,
                          acc.V3.x, acc.V3.y, acc.v22, (float)acc.cnt, acc.s0f};
#pragma unroll
    for (int k = 0; k < 11; ++k) v[36 + k] = group_sumf<L>(vv[k]);
    const double l1 = kL1 ? group_sum<L>(acc.l1) : 0.0;
    if (has_item) {
#pragma unroll
      for (int vi = 0; vi < 47; ++vi) {
        if (vi % L != g) continue;
        if (vi == 46) {
          if (single) out.s0[d.n] = (double)v[vi];
          else part.s0[item] = (double)v[vi];
          continue;
        }
        const int k = hot_out_index(vi);
        if (k >= 0) store_red(out, part, single, P, NI, d.n, item, k, v[vi], kLin);
      }
      if (kL1 && g == 0) {
        if (single) {
          if (out.l1) out.l1[d.n] = l1;
        } else {
          part.l1[item] = l1;
        }
      }
    }
  } else {
    const int cnt = (int)group_sum<L>((double)acc.cnt);
    const double l1 = kL1 ? group_sum<L>(acc.l1) : 0.0;
    if (has_item && g == 0) {
      if (single) {
        if (out.n_active) out.n_active[d.n] = cnt;
        if (kL1 && out.l1) out.l1[d.n] = l1;
      } else {
        static_cast<float*>(part.red)[45 * NI + item] = (float)cnt;
        if (kL1) part.l1[item] = l1;
      }
    }
  }
}

// -------------------------------------------------------------- generic kernel
// API modes: optional z columns, fp64 moments, caller-given residual weights,
// residual output, mask-free sweeps.  Plain scalar code; not on the hot loop.
template <bool HOMOG, bool F64, unsigned MODE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
point_pass_generic(const fm_point_store s, const double* __restrict__ ghat,
                   const double* __restrict__ res_in, const double thr,
                   const int32_t* __restrict__ prev_active, const fm_pass_out out,
                   const PartialBufs part) {
  using Acc = typename std::conditional<F64, double, float>::type;
  constexpr bool kPrune = MODE & FM_PASS_PRUNE;
  constexpr bool kL1 = MODE & FM_PASS_L1;
  constexpr bool kMom = MODE & FM_PASS_MOMENTS;
  constexpr bool kIrls = MODE & FM_PASS_IRLS;
  constexpr bool kAll = MODE & FM_PASS_ALL_POINTS;
  constexpr bool kResOut = MODE & FM_PASS_RES_OUT;
  constexpr bool kResIn = MODE & FM_PASS_RES_IN;
  constexpr bool kSkip = MODE & FM_PASS_SKIP_DROPPED;
  constexpr bool kNeedR = kPrune || kL1 || kIrls || kResOut;
  constexpr bool kLin = kMom && kIrls;

  const int lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (item >= s.n_items) return;
  const int n = s.item_pair[item];
  const int first = s.pair_item_off[n];
  const bool single = (s.pair_item_off[n + 1] - first) == 1;
  const int64_t P = s.n_pairs;

  Acc mom[36], vg[9];
#pragma unroll
  for (int k = 0; k < 36; ++k) mom[k] = Acc(0);
#pragma unroll
  for (int k = 0; k < 9; ++k) vg[k] = Acc(0);
  double s0 = 0.0, l1 = 0.0;
  int cnt = 0;

  if (!(kSkip && prev_active[n] == 0)) {
    double G[9];
    if (kNeedR) {
#pragma unroll
      for (int k = 0; k < 9; ++k) G[k] = ghat[k * P + n];
    }
    const int64_t base = s.pair_off[n];
    const int64_t end = base + s.pair_len[n];
    const int64_t lo = base + (int64_t)(item - first) * s.chunk;
    const int64_t hi = end < lo + s.chunk ? end : lo + s.chunk;
    for (int64_t cb = lo + 4 * lane; cb < hi; cb += 128) {
      const int shift = (int)(cb & 31);
      const unsigned bits = kAll ? 0xFu : ((s.active[cb >> 5] >> shift) & 0xFu);
      unsigned keep_bits = 0;
      for (int k = 0; k < 4; ++k) {
        const int64_t sl = cb + k;
        const bool valid = sl < hi;
        const bool act = valid && ((bits >> k) & 1u);
        if (!valid) continue;
        const double a = s.x1[2 * sl], bb = s.x1[2 * sl + 1];
        const double c = s.x2[2 * sl], d = s.x2[2 * sl + 1];
        const double e = HOMOG ? (double)s.x1z[sl] : 1.0;
        const double f = HOMOG ? (double)s.x2z[sl] : 1.0;
        double r = 0.0;
        if (kNeedR) {
          const double y0 = fma(G[0], a, fma(G[1], bb, G[2] * e));
          const double y1 = fma(G[3], a, fma(G[4], bb, G[5] * e));
          const double y2 = fma(G[6], a, fma(G[7], bb, G[8] * e));
          r = fma(c, y0, fma(d, y1, f * y2));
        }
        const double ar = fabs(r);
        if (kResOut) out.residual[sl] = ar;
        const bool keep = kPrune ? (act && ar <= thr) : act;
        keep_bits |= (unsigned)keep << k;
        cnt += keep;
        if (kL1) l1 += act ? ar : 0.0;
        if (kMom && keep) {
          double w = 1.0;
          if (kIrls) w = 1.0 / fmax(ar, 1e-6);
          else if (kResIn) w = 1.0 / fmax(fabs(res_in[sl]), 1e-6);
          const double A6[6] = {a * a, a * bb, a * e, bb * bb, bb * e, e * e};
          const double wc = w * c, wd = w * d, wf = w * f;
          const double B6[6] = {wc * c, wc * d, wc * f, wd * d, wd * f, wf * f};
#pragma unroll
          for (int i = 0; i < 6; ++i)
#pragma unroll
            for (int j = 0; j < 6; ++j) mom[i * 6 + j] += Acc(B6[i] * A6[j]);
          if (kLin) {
            const double wr = w * r;
            s0 += wr * r;
            const double x2v[3] = {wr * c, wr * d, wr * f};
            const double x1v[3] = {a, bb, e};
#pragma unroll
            for (int p = 0; p < 3; ++p)
#pragma unroll
              for (int q = 0; q < 3; ++q) vg[p * 3 + q] += Acc(x2v[p] * x1v[q]);
          }
        }
      }
      if (kPrune) {
        const unsigned cleared = bits & ~keep_bits & 0xFu;
        if (cleared) atomicAnd(&s.active[cb >> 5], ~(cleared << shift));
      }
    }
  }

  if (kMom) {
    Acc v[64];
#pragma unroll
    for (int k = 0; k < 36; ++k) v[k] = mom[k];
#pragma unroll
    for (int k = 0; k < 9; ++k) v[36 + k] = vg[k];
    v[45] = Acc(cnt);
#pragma unroll
    for (int k = 46; k < 64; ++k) v[k] = Acc(0);
    warp_transpose_reduce64(v, lane);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int k = 2 * lane + h;
      if (k >= kNumRed) continue;
      if (!single) {
        static_cast<Acc*>(part.red)[k * s.n_items + item] = v[h];
      } else if (k < 36) {
        if (F64) out.mom64[k * P + n] = (double)v[h];
        else out.mom32[k * P + n] = (float)v[h];
      } else if (k < 45) {
        if (kLin && out.vgrad) out.vgrad[(k - 36) * P + n] = (float)v[h];
      } else if (out.n_active) {
        out.n_active[n] = (int32_t)v[h];
      }
    }
  } else {
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if (lane == 0) {
      if (!single) static_cast<Acc*>(part.red)[45 * s.n_items + item] = Acc(cnt);
      else if (out.n_active) out.n_active[n] = cnt;
    }
  }
  if (kLin) {
    s0 = warp_sum(s0);
    if (lane == 0) {
      if (single) { if (out.s0) out.s0[n] = s0; }
      else part.s0[item] = s0;
    }
  }
  if (kL1) {
    l1 = warp_sum(l1);
    if (lane == 0) {
      if (single) { if (out.l1) out.l1[n] = l1; }
      else part.l1[item] = l1;
    }
  }
}

// Sum the partials of pairs split over several work items, in item order.
template <bool F64, unsigned MODE>
__global__ void combine_kernel(const fm_point_store s, const fm_pass_out out,
                               const PartialBufs part, const bool has_lin) {
  using Acc = typename std::conditional<F64, double, float>::type;
  constexpr bool kL1 = MODE & FM_PASS_L1;
  constexpr bool kMom = MODE & FM_PASS_MOMENTS;
  const bool kLin = kMom && (MODE & FM_PASS_IRLS) && has_lin;
  const int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= s.n_pairs) return;
  const int i0 = s.pair_item_off[n], i1 = s.pair_item_off[n + 1];
  if (i1 - i0 <= 1) return;
  const int64_t P = s.n_pairs, NI = s.n_items;
  const Acc* red = static_cast<const Acc*>(part.red);
  for (int k = kMom ? 0 : 45; k < kNumRed; ++k) {
    Acc acc = 0;
    if (k >= 36 && k < 45 && !kLin) continue;
    for (int i = i0; i < i1; ++i) acc += red[k * NI + i];
    if (k < 36) {
      if (F64) out.mom64[k * P + n] = (double)acc;
      else out.mom32[k * P + n] = (float)acc;
    } else if (k < 45) {
      if (kLin && out.vgrad) out.vgrad[(k - 36) * P + n] = (float)acc;
    } else if (out.n_active) {
      out.n_active[n] = (int32_t)acc;
    }
  }
  if (kLin && out.s0) {
    double acc = 0;
    for (int i = i0; i < i1; ++i) acc += part.s0[i];
    out.s0[n] = acc;
  }
  if (kL1 && out.l1) {
    double acc = 0;
    for (int i = i0; i < i1; ++i) acc += part.l1[i];
    out.l1[n] = acc;
  }
}

template <unsigned MODE, bool MOM64, int L>
int hot_blocks_per_sm(int* out) {
  static int cached = 0;
  if (!cached) {
    const size_t smem = kGrpWarps * sizeof(LaneRing);
    FM_CUDA(cudaFuncSetAttribute(point_pass_hot<MODE, MOM64, L>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int b = 0;
    FM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, point_pass_hot<MODE, MOM64, L>,
                                                          kGrpWarps * 32, smem));
    cached = b > 0 ? b : 1;
  }
  *out = cached;
  return FM_OK;
}

template <unsigned MODE, bool MOM64, int L>
int launch_hot_l(const fm_point_store& s, double thr, const double* ghat, const int32_t* prev_active,
                 const fm_pass_out& out, const PartialBufs& part, cudaStream_t stream) {
  const size_t smem = kGrpWarps * sizeof(LaneRing);
  const int64_t warps = ceil_div(s.n_items, 32 / L);
  const int64_t grid = ceil_div(warps, kGrpWarps);
  point_pass_hot<MODE, MOM64, L><<<(unsigned)grid, kGrpWarps * 32, smem, stream>>>(
      s, ghat, thr, prev_active, out, part);
  FM_LAUNCHED(point_pass_hot);
  if (s.n_items > s.n_pairs) {
    combine_kernel<MOM64, MODE><<<(unsigned)ceil_div(s.n_pairs, 128), 128, 0, stream>>>(s, out, part,
                                                                                        !MOM64);
    FM_LAUNCHED(combine_kernel);
  }
  return FM_OK;
}

// Lanes per item L: blocks are one-shot, so the last wave of a launch is
// partially filled.  Score each L by (work / slots-time) of its wave count
// and a per-item reduction cost of log2(L) butterfly levels; short items
// (< 4L slots per lane-iteration) also waste lanes.
template <unsigned MODE, bool MOM64>
int launch_hot(const fm_point_store& s, double thr, const double* ghat, const int32_t* prev_active,
               const fm_pass_out& out, const PartialBufs& part, cudaStream_t stream) {
  int b4 = 1, b8 = 1, b16 = 1;
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 4>(&b4)) return rc;
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 8>(&b8)) return rc;
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 16>(&b16)) return rc;
  const double mean_len = s.n_items ? (double)s.n_slots / (double)s.n_items : 0.0;
  const int Ls[3] = {4, 8, 16};
  const int bps[3] = {b4, b8, b16};
  double best = -1.0;
  int pick = 4;
  for (int k = 0; k < 3; ++k) {
    const int L = Ls[k];
    const double blocks = std::ceil((double)s.n_items / (32.0 / L) / kGrpWarps);
    const double resident = (double)bps[k] * sm_count();
    const double waves = blocks / resident;
    const double fill = waves / std::ceil(waves);
    const double lane_use = std::min(1.0, mean_len / (4.0 * L)) ;
    const double red = 1.0 / (1.0 + 0.02 * (k + 2) * 400.0 / std::max(mean_len, 1.0));
    const double score = fill * lane_use * red;
    if (score > best * 1.03) {
      best = score;
      pick = L;
    }
  }
  if (const char* env = getenv("FM_HOT_L")) pick = atoi(env);  // tuning override
  if (pick == 16) return launch_hot_l<MODE, MOM64, 16>(s, thr, ghat, prev_active, out, part, stream);
  if (pick == 8) return launch_hot_l<MODE, MOM64, 8>(s, thr, ghat, prev_active, out, part, stream);
  return launch_hot_l<MODE, MOM64, 4>(s, thr, ghat, prev_active, out, part, stream);
}

template <bool HOMOG, bool F64, unsigned MODE>
int launch_generic(const fm_point_store& s, double thr, const double* ghat, const double* res_in,
                   const int32_t* prev_active, const fm_pass_out& out, const PartialBufs& part,
                   cudaStream_t stream) {
  const int64_t blocks = ceil_div(s.n_items, kWarpsPerBlock);
  point_pass_generic<HOMOG, F64, MODE><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, stream>>>(
      s, ghat, res_in, thr, prev_active, out, part);
  FM_LAUNCHED(point_pass_generic);
  if (s.n_items > s.n_pairs) {
    combine_kernel<F64, MODE><<<(unsigned)ceil_div(s.n_pairs, 128), 128, 0, stream>>>(s, out, part,
                                                                                      true);
    FM_LAUNCHED(combine_kernel);
  }
  return FM_OK;
}

constexpr unsigned kSkipD = FM_PASS_SKIP_DROPPED;
constexpr unsigned kIrlsM = FM_PASS_MOMENTS | FM_PASS_IRLS;

// Hot combinations (z == 1): the passes of irls_refine (rounds 0 / 1+,
// IRLS iterations, final L1) and the API's L1 loss.
#define FM_HOT_MODES(X)                                  \
  X(FM_PASS_PRUNE | kIrlsM)                              \
  X(FM_PASS_L1 | FM_PASS_PRUNE | kIrlsM)                 \
  X(FM_PASS_L1 | FM_PASS_PRUNE | kIrlsM | kSkipD)        \
  X(kIrlsM | kSkipD)                                     \
  X(FM_PASS_L1)                                          \
  X(FM_PASS_L1 | kSkipD)

// Generic combinations (API functions, any z, fp32 or fp64 accumulation).
#define FM_GENERIC_MODES(X)                                          \
  FM_HOT_MODES(X)                                                    \
  X(FM_PASS_PRUNE | kIrlsM | kSkipD)                                 \
  X(kIrlsM)                                                          \
  X(FM_PASS_PRUNE)                                                   \
  X(FM_PASS_PRUNE | kSkipD)                                          \
  X(FM_PASS_ALL_POINTS | FM_PASS_RES_OUT)                            \
  X(FM_PASS_MOMENTS)                                                 \
  X(FM_PASS_MOMENTS | FM_PASS_ALL_POINTS)                            \
  X(FM_PASS_MOMENTS | FM_PASS_ALL_POINTS | FM_PASS_RES_IN)           \
  X(FM_PASS_MOMENTS | FM_PASS_RES_IN)                                \
  X(FM_PASS_MOMENTS | FM_PASS_L1)

template <bool HOMOG, bool F64>
int dispatch_generic(unsigned mode, const fm_point_store& s, double thr, const double* ghat,
                     const double* res_in, const int32_t* prev_active, const fm_pass_out& out,
                     const PartialBufs& part, cudaStream_t stream) {
#define FM_CASE(M) \
  if (mode == (M)) return launch_generic<HOMOG, F64, (M)>(s, thr, ghat, res_in, prev_active, out, part, stream);
  FM_GENERIC_MODES(FM_CASE)
#undef FM_CASE
  return set_error(FM_ERR_INVALID, "unsupported point-pass mode 0x%x", mode);
}

int dispatch_hot(unsigned mode, bool f64, const fm_point_store& s, double thr, const double* ghat,
                 const int32_t* prev_active, const fm_pass_out& out, const PartialBufs& part,
                 cudaStream_t stream, bool* handled) {
  *handled = true;
  if (f64) {
#define FM_CASE(M) \
  if (mode == (M)) return launch_hot<(M), true>(s, thr, ghat, prev_active, out, part, stream);
    FM_HOT_MODES(FM_CASE)
#undef FM_CASE
  } else {
#define FM_CASE(M) \
  if (mode == (M)) return launch_hot<(M), false>(s, thr, ghat, prev_active, out, part, stream);
    FM_HOT_MODES(FM_CASE)
#undef FM_CASE
  }
  *handled = false;
  return FM_OK;
}

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

size_t fm_point_pass_scratch_bytes(const fm_point_store* store) {
  if (!store) return 0;
  const size_t ni = (size_t)store->n_items;
  return scratch_round(ni * kNumRed * sizeof(double)) + 2 * scratch_round(ni * sizeof(double)) +
         scratch_round(ni * 4 * sizeof(int32_t)) + 256;
}

int fm_point_store_describe(const fm_point_store* store, void* stream) {
  FM_REQUIRE(store && store->item_desc, "null store or item_desc");
  if (store->n_items == 0) return FM_OK;
  describe_items_kernel<<<(unsigned)ceil_div(store->n_items, 256), 256, 0, as_stream(stream)>>>(
      *store, store->item_desc);
  FM_LAUNCHED(describe_items_kernel);
  return FM_OK;
}

int fm_point_pass(const fm_point_store* store, unsigned mode, double threshold, const double* ghat,
                  const double* res_in, const int32_t* prev_active, const fm_pass_out* out,
                  void* scratch, size_t scratch_bytes, void* stream) {
  FM_REQUIRE(store && out, "null store/out");
  const fm_point_store& s = *store;
  FM_REQUIRE(s.n_pairs >= 0 && s.n_items >= s.n_pairs && s.chunk > 0 && s.chunk % 128 == 0,
             "bad store geometry (pairs=%lld items=%lld chunk=%lld)", (long long)s.n_pairs,
             (long long)s.n_items, (long long)s.chunk);
  FM_REQUIRE(s.n_slots % 128 == 0, "n_slots must be a multiple of 128");
  if (s.n_pairs == 0) return FM_OK;
  FM_REQUIRE(s.x1 && s.x2 && s.active && s.pair_off && s.pair_len && s.pair_item_off && s.item_pair,
             "incomplete point store");
  FM_REQUIRE(((uintptr_t)s.x1 % 16) == 0 && ((uintptr_t)s.x2 % 16) == 0,
             "coordinate columns must be 16-byte aligned");
  const bool homog = s.x1z != nullptr;
  FM_REQUIRE(homog == (s.x2z != nullptr), "x1z and x2z must both be set or both NULL");
  const bool f64 = (mode & FM_PASS_F64) != 0;
  const unsigned m = mode & ~FM_PASS_F64;
  const bool need_r = m & (FM_PASS_PRUNE | FM_PASS_L1 | FM_PASS_IRLS | FM_PASS_RES_OUT);
  FM_REQUIRE(!need_r || ghat, "mode 0x%x needs ghat", mode);
  FM_REQUIRE(!(m & FM_PASS_RES_IN) || res_in, "FM_PASS_RES_IN needs res_in");
  FM_REQUIRE(!(m & FM_PASS_RES_OUT) || out->residual, "FM_PASS_RES_OUT needs out->residual");
  FM_REQUIRE(!(m & FM_PASS_SKIP_DROPPED) || prev_active, "SKIP_DROPPED needs prev_active");
  if (m & FM_PASS_MOMENTS) {
    FM_REQUIRE(f64 ? out->mom64 != nullptr : out->mom32 != nullptr, "moment output missing");
    if ((m & FM_PASS_IRLS) && !f64) FM_REQUIRE(out->vgrad && out->s0, "IRLS pass needs vgrad/s0");
  }
  PartialBufs part{nullptr, nullptr, nullptr};
  cudaStream_t st = as_stream(stream);
  fm_point_store s2 = s;  // with item descriptors
  {
    Scratch sc(scratch, scratch_bytes);
    if (s.n_items > s.n_pairs) {
      part.red = sc.take<double>((size_t)s.n_items * kNumRed);
      part.s0 = sc.take<double>((size_t)s.n_items);
      part.l1 = sc.take<double>((size_t)s.n_items);
    }
    if (!s.item_desc) {
      s2.item_desc = sc.take<int32_t>((size_t)s.n_items * 4);
      if (int rc = fm_point_store_describe(&s2, stream)) return rc;
    }
    FM_REQUIRE((sc.used == 0 || scratch) && sc.ok(), "point-pass scratch too small (%zu < %zu)",
               scratch_bytes, sc.used);
  }
  if (!homog) {
    // fp64 moments are the exact default; fp32 (FFMA2 + shifted model) only for IRLS moments
    const bool hot_f64 = f64 || !(m & FM_PASS_MOMENTS);
    bool handled = false;
    if (hot_f64 || (m & FM_PASS_IRLS)) {
      const int rc = dispatch_hot(m, hot_f64, s2, threshold, ghat, prev_active, *out, part, st, &handled);
      if (handled) return rc;
    }
  }
  if (homog) {
    return f64 ? dispatch_generic<true, true>(m, s, threshold, ghat, res_in, prev_active, *out, part, st)
               : dispatch_generic<true, false>(m, s, threshold, ghat, res_in, prev_active, *out, part, st);
  }
  return f64 ? dispatch_generic<false, true>(m, s, threshold, ghat, res_in, prev_active, *out, part, st)
             : dispatch_generic<false, false>(m, s, threshold, ghat, res_in, prev_active, *out, part, st);
}

}  // extern "C"
