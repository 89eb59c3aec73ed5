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

// Exact pass totals: kTotSlots copies of the integer accumulators (a warp
// adds into copy wid % kTotSlots, so same-address reductions do not pile up)
constexpr int kTotSlots = 64;
struct TotSlot {
  unsigned long long l1_int, l1_f1, l1_f2;  // fixed-point L1: int + 2^-32 + 2^-64 words
  unsigned long long z, kept;
  unsigned flags;  // 1: NaN L1, 2: +inf L1
  unsigned pad;
};
struct TotCtl {  // zero-initialised scratch, re-armed after every launch
  TotSlot slot[kTotSlots];
};

struct PartialBufs {
  void* red;   // [kNumRed][n_items] of the accumulator type
  double* s0;  // [n_items]
  double* l1;  // [n_items]
  int64_t cap; // items the buffers hold
  double* tot_part;  // per-block partials of fm_pass_totals (generic / chunked passes)
  double* totals;
  TotCtl* ctl;  // fused totals of the one-shot hot kernel (exact integer sums)
};

// Converts the exact sums of the launch before it into `totals` and re-arms
// the control words.  Launched right after the pass as a programmatic
// dependent launch: it is scheduled while the pass drains and waits for the
// pass's completion and memory flush in griddepcontrol.wait.
__global__ void totals_finalize_kernel(TotCtl* c, double* totals) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  static_assert(kTotSlots == 64, "two slots per lane");
  const int lane = threadIdx.x;
  unsigned long long v[5];
  unsigned fl = 0;
#pragma unroll
  for (int k = 0; k < 5; ++k) v[k] = 0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    TotSlot& t = c->slot[lane + 32 * q];
    v[0] += t.l1_int; v[1] += t.l1_f1; v[2] += t.l1_f2; v[3] += t.z; v[4] += t.kept;
    fl |= t.flags;
    t.l1_int = t.l1_f1 = t.l1_f2 = t.z = t.kept = 0ull;
    t.flags = 0u;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < 5; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    fl |= __shfl_xor_sync(0xffffffffu, fl, off);
  }
  if (lane != 0) return;
  if (totals) {
    double l1 = (double)v[0] + ldexp((double)v[1], -32) + ldexp((double)v[2], -64);
    if (fl & 1u) l1 = __longlong_as_double(0x7ff8000000000000ll);
    else if (fl & 2u) l1 = __longlong_as_double(0x7ff0000000000000ll);
    totals[0] = l1;
    totals[1] = (double)v[3];
    totals[2] = (double)v[4];
  }
}

int launch_totals_finalize(TotCtl* c, double* totals, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = getenv("FM_NO_PDL") ? 0 : 1;
  FM_CUDA(cudaLaunchKernelEx(&cfg, totals_finalize_kernel, c, totals));
  FM_LAUNCHED(totals_finalize_kernel);
  return FM_OK;
}

// Exact, order-independent pass totals: a warp adds its items' {L1, Z, kept}
// with fire-and-forget integer reductions (no fence, no ticket: a block-exit
// fence + atomic ticket cost ~3 us at C2 by delaying every block's
// retirement); L1 is cut into an integer part and two 32-bit fraction words,
// exact for the double, so the sum does not depend on the order the warps
// finish in and the pass stays bitwise reproducible.
__device__ __forceinline__ void totals_add(TotCtl* ctl, unsigned wid, double l1, double z,
                                           double kept) {
  TotSlot* c = &ctl->slot[wid % kTotSlots];
  if (isfinite(l1)) {
    const double ip = floor(l1);
    const double f1 = ldexp(l1 - ip, 32);
    const double f1i = floor(f1);
    const double f2 = floor(ldexp(f1 - f1i, 32));
    atomicAdd(&c->l1_int, (unsigned long long)ip);
    atomicAdd(&c->l1_f1, (unsigned long long)f1i);
    atomicAdd(&c->l1_f2, (unsigned long long)f2);
  } else {
    atomicOr(&c->flags, isnan(l1) ? 1u : 2u);
  }
  atomicAdd(&c->z, (unsigned long long)z);
  atomicAdd(&c->kept, (unsigned long long)kept);
}


#ifdef FM_HOT_TRACE
// Tuning build only: per-block {smid, start ns, end ns, items} of the last hot launch.
__device__ unsigned long long g_hot_trace[16384][4];
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif



// ------------------------------------------------------------------ hot kernel
// z == 1 stores whose pairs start on 16-slot boundaries (store->slot_align
// >= 16; the slots between a pair's last point and the next boundary are
// inactive padding).  Every work item is then a whole number of 16-slot
// blocks, so the loop carries no per-slot bounds checks: the active mask alone
// says which slots count.
//
// A warp works on 32/L consecutive work items at once: L lanes per item
// (L in {4, 8}).  Iteration `it` of a lane group covers the 16-slot block at
// item.lo + 16*it; lane g owns the 16-byte chunks c = g + L*j (j < 8/L) of
// each coordinate column, i.e. slots {2c, 2c+1} of the block, so each copy
// instruction of a group reads whole 32-byte sectors.  The chunks stream
// through a private per-lane ring of kRing shared-memory stages filled with
// cp.async (LDGSTS, L2-only 16-byte copies, one commit group per iteration):
// every lane reads back only what it copied itself, so cp.async.wait_group
// suffices (no barriers).  Per-item totals need log2(L) butterfly levels
// across the item's lanes (fixed order -> bitwise reproducible).
//
// Per point pair: the fp64 residual r = x2^T Ghat x1 (8 DFMA on converted
// coordinates), the prune decision |r| <= th in fp64, the pre-prune L1 in
// fp64, the IRLS weight 1/max(|r|, 1e-6) (fp32 reciprocal of the rounded
// residual: a per-point relative error keeps every term rank-1 exact) masked
// by the post-prune keep bit, and the 36 Kronecker moments
//   mom[i][j] = sum w B_i A_j,  B = (c^2, cd, c, d^2, d, 1),
//                               A = (a^2, ab, a, b^2, b, 1)
// for x1 = (a, b), x2 = (c, d).
// MOM64 = true (exact): the moments accumulate in fp64 (36 DFMA / point).
// MOM64 = false (fast): fp32 moments in the "B-pair" form -- each A_j is a
// scalar broadcast against the three natural float2 pairs
//   (w c^2, w d^2) = (w c, w d) * (c, d),  (w c, w d),  (w c d, w)
// so 15 packed FFMA2 + 3 FADD2 cover the 36 moments -- plus the shifted-model
// linearisation terms vgrad = sum w r t and s0 = sum w r^2.
#ifndef FM_HOT_RING
#define FM_HOT_RING 4
#endif
#ifndef FM_HOT_UNROLL
#define FM_HOT_UNROLL 1
#endif
#ifndef FM_SHORT_RING
#define FM_SHORT_RING 3  // ring stages of short mixed launches (see launch_hot)
#endif
#ifndef FM_HOT_MINB
#define FM_HOT_MINB 4
#endif
#ifndef FM_HOT_MINB64
#define FM_HOT_MINB64 3
#endif
constexpr int kRing = FM_HOT_RING;  // stages per lane
constexpr int kUnroll = FM_HOT_UNROLL;  // main-loop unroll (points in flight per lane = 4 x kUnroll)
#ifndef FM_GRP_WARPS
#define FM_GRP_WARPS 4
#endif
constexpr int kGrpWarps = FM_GRP_WARPS;  // warps per block (2, 8 or 16: slower, measured)
constexpr int kBlkSlots = 16;       // slots per group iteration (= slot alignment)

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

#ifndef FM_HOT_NOLOAD
#define FM_HOT_NOLOAD 0  // tuning experiment only: skip the coordinate/mask copies
#endif
template <bool kPrune, bool kL1, bool kMom, bool MOM64>
struct HotAcc {
  double M64[MOM64 ? 36 : 1];
  float2 Mp[MOM64 ? 1 : 18];  // [j][k]: A_j x B-pair k, k: (B0,B3) (B2,B4) (B1,B5)
  float2 V0, V1, V2, V3;      // (v00,v01) (v10,v11) (v20,v21) (v02,v12)
  float v22, s0f;
  double l1;
  float l1f;
  int cnt;

  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int k = 0; k < (MOM64 ? 36 : 1); ++k) M64[k] = 0.0;
#pragma unroll
    for (int k = 0; k < (MOM64 ? 1 : 18); ++k) Mp[k] = f2(0.f);
    V0 = V1 = V2 = V3 = f2(0.f);
    v22 = s0f = 0.f;
    l1 = 0.0;
    l1f = 0.f;
    cnt = 0;
  }

  // One point pair; returns the post-prune keep flag.  Branch-free: the
  // residual and weight are computed for every slot and masked afterwards.
  __device__ __forceinline__ bool point(const double (&G)[9], float a, float b, float c, float d,
                                        bool act, double thr) {
    // residual r = x2^T Ghat x1 in fp64 (ref/epipolar.py:255)
    const double A = a, B = b, C = c, D = d;
    const double y0 = fma(G[0], A, fma(G[1], B, G[2]));
    const double y1 = fma(G[3], A, fma(G[4], B, G[5]));
    const double y2 = fma(G[6], A, fma(G[7], B, G[8]));
    const double r = fma(C, y0, fma(D, y1, y2));
    const double ar = fabs(r);
    const bool keep = (kPrune && !FM_HOT_NOLOAD) ? (act & (ar <= thr)) : act;
    // fp32 moment passes sum L1 in fp32 from the rounded residual (per-lane
    // partials of ~10^2 terms, relative error ~1e-6; fp64 across lanes)
    const float rf = (float)r;
    if (kL1 && kMom && !MOM64) l1f += act ? fabsf(rf) : 0.f;
    else if (kL1) l1 += act ? ar : 0.0;
    if (!kMom) return keep;
    // IRLS weight 1/max(|r|, 1e-6) (ref/epipolar.py:58); the opaque AND (not a
    // select) keeps the reciprocal out of a per-point branch.  Coordinates of
    // every slot are finite (store builders zero and deactivate non-finite
    // points), so w = +0 removes a dropped point exactly.
    const float w = and_mask(rcp_approx(fmaxf(fabsf(rf), 1e-6f)), keep ? 0xffffffffu : 0u);
    if (MOM64) {
      const double wd = w;
      const double p = wd * C, q = wd * D;
      const double Bv[6] = {p * C, p * D, p, q * D, q, wd};
      const double Av[5] = {A * A, A * B, A, B * B, B};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
#pragma unroll
        for (int j = 0; j < 5; ++j) M64[MOM64 ? i * 6 + j : 0] = fma(Bv[i], Av[j], M64[MOM64 ? i * 6 + j : 0]);
        M64[MOM64 ? i * 6 + 5 : 0] += Bv[i];
      }
    } else {
      const float2 X1 = make_float2(a, b), X2 = make_float2(c, d);
      const float2 PQ = __fmul2_rn(f2(w), X2);         // (w c, w d)
      const float2 Bp[3] = {__fmul2_rn(PQ, X2),        // (w c^2, w d^2)
                            PQ,                        // (w c, w d)
                            make_float2(PQ.x * d, w)}; // (w c d, w)
      const float2 AA = __fmul2_rn(f2(a), X1);         // (a^2, a b)
      const float Av[5] = {AA.x, AA.y, a, b * b, b};
#pragma unroll
      for (int j = 0; j < 5; ++j)
#pragma unroll
        for (int k = 0; k < 3; ++k)
          Mp[MOM64 ? 0 : j * 3 + k] = __ffma2_rn(f2(Av[j]), Bp[k], Mp[MOM64 ? 0 : j * 3 + k]);
#pragma unroll
      for (int k = 0; k < 3; ++k) Mp[MOM64 ? 0 : 15 + k] = __fadd2_rn(Bp[k], Mp[MOM64 ? 0 : 15 + k]);
      // shifted-model terms: w r0 (= sign(r0) unless clamped), w r0^2
      const float wr = w * rf;
      s0f = fmaf(wr, rf, s0f);
      const float2 S = __fmul2_rn(f2(wr), X2);
      V0 = __ffma2_rn(f2(S.x), X1, V0);
      V1 = __ffma2_rn(f2(S.y), X1, V1);
      V2 = __ffma2_rn(f2(wr), X1, V2);
      V3 = __fadd2_rn(S, V3);
      v22 += wr;
    }
    return keep;
  }
};

// Canonical moment index (row i = B, column j = A) of hot fp32 slot v (0..35):
// slot v = 2 (3 j + k) + h holds B-pair k's half h against A_j, and the
// B-pairs are (B0, B3), (B2, B4), (B1, B5).
__device__ __forceinline__ int hot_mom_index(int v) {
  const int m = v >> 1, h = v & 1;
  const int j = m / 3, k = m - 3 * j;
  const int row = k == 0 ? 3 * h : (k == 1 ? 2 + 2 * h : 1 + 4 * h);
  return row * 6 + j;
}

template <int L>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
  for (int off = 1; off < L; off <<= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}

// Transpose-reduce of N values (N % L == 0) across the L lanes of an aligned
// lane group: every level halves the values a lane carries (it keeps one half,
// sends the other to its partner), so log2(L) levels cost N/2 + N/4 + ...
// shuffles instead of N log2(L).  Afterwards lane g of the group holds the
// group sums of values [g N/L, (g+1) N/L) in v[0 .. N/L).  Fixed order ->
// bitwise reproducible.
template <int L, int N, typename T>
__device__ __forceinline__ void group_transpose_reduce(T (&v)[N], int lane) {
  static_assert(N % L == 0, "N must be a multiple of L");
#pragma unroll
  for (int lvl = 0; (1 << lvl) < L; ++lvl) {
    const int o = L >> (lvl + 1);
    const int half = N >> (lvl + 1);
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const T send = upper ? v[i] : v[i + half];
      const T keep = upper ? v[i + half] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// Per-lane ring: stage d holds the lane's two chunks of x1 then of x2
// (chunk-major: a warp's LDS.128 of one chunk row touches 32 consecutive
// 16-byte words) and the mask word of the lane's block.
// Stage-major: a lane's mask slot sits at a fixed (per-lane) distance from its
// chunk slots in the same stage, so one running stage address serves the
// copies, the chunk reads and the mask read (no per-iteration stage index
// arithmetic).
struct LaneStage {
  float4 c[4][32];
  uint32_t m[32];
};
template <int RING>
struct LaneRingT {
  LaneStage s[RING];
};
using LaneRing = LaneRingT<kRing>;

// L = 4 S lanes per work item: S sub-groups of 4 lanes; iteration `it`
// covers blocks S*it .. S*it + S - 1 of the item, sub-group sg takes block
// S*it + sg, and its lane h the 16-byte chunks h and h + 4 of each column
// (slots {2h, 2h+1, 2h+8, 2h+9}): every copy instruction of a sub-group reads
// whole 32-byte sectors.
template <unsigned MODE, bool MOM64, int L, int RING = kRing>
__device__ __forceinline__ void hot_body(const fm_point_store& s, const double* __restrict__ ghat,
                                         const double thr, const int32_t* __restrict__ prev_active,
                                         const fm_pass_out& out, const PartialBufs& part,
                                         const int64_t group, const int64_t item_base,
                                         const int64_t item_end) {
  constexpr bool kPrune = MODE & FM_PASS_PRUNE;
  constexpr bool kL1 = MODE & FM_PASS_L1;
  constexpr bool kMom = (MODE & FM_PASS_MOMENTS) && (MODE & FM_PASS_IRLS);
  constexpr bool kLin = kMom && !MOM64;
  constexpr bool kSkip = MODE & FM_PASS_SKIP_DROPPED;
  constexpr int IPW = 32 / L;  // items per warp
  constexpr int S = L / 4;     // blocks per iteration
  static_assert(L == 4 || L == 8 || L == 16 || L == 32, "L in {4, 8, 16, 32}");

  if (out.stop && *out.stop) return;  // an earlier stage failed: leave everything alone
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  LaneRingT<RING>& ring = reinterpret_cast<LaneRingT<RING>*>(smem_raw)[wib];
#ifdef FM_HOT_TRACE
  const unsigned long long t_start = globaltimer();
#endif
  const int64_t P = s.n_pairs;
  const int g = lane % L;  // lane within the item group
  const int sg = g >> 2;   // sub-group: block offset within an iteration
  const int h = g & 3;     // lane within the sub-group
  const int64_t item = item_base + group * IPW + lane / L;  // group: the warp's item group
  const bool has_item = item < item_end;  // item_end <= n_items
  const int64_t NI = s.n_items;

  ItemDesc d{0, 0, 0, true};
  if (has_item) d = decode_item(__ldg(reinterpret_cast<const int4*>(s.item_desc) + item));
  // one item per pair (the common case): item == pair, so the pair loads need
  // not wait for the descriptor (one dependent global-load latency less)
  const int64_t pn = (NI == P) ? item : d.n;
  const bool skip = has_item && kSkip && __ldg(prev_active + pn) == 0;
  double G[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) G[k] = has_item ? __ldg(ghat + k * P + pn) : 0.0;
  const int nblk = (has_item && !skip) ? (d.len + kBlkSlots - 1) / kBlkSlots : 0;  // skipped: no work
  const int nit = (nblk + S - 1) / S;
  const int warp_it = __reduce_max_sync(0xffffffffu, nit);

  // 16 slots = 128 B = 8 float4 per column per block
  const float4* x1b = reinterpret_cast<const float4*>(s.x1 + 2 * d.lo) + 8 * sg + h;
  const float4* x2b = reinterpret_cast<const float4*>(s.x2 + 2 * d.lo) + 8 * sg + h;
  const int half0 = (int)(d.lo & 16) + kBlkSlots * sg;  // bit of block sg relative to word lo/32
  const uint32_t* mwb = reinterpret_cast<const uint32_t*>(s.active) + (d.lo >> 5);
  uint32_t* mwb_w = reinterpret_cast<uint32_t*>(s.active) + (d.lo >> 5);

  constexpr uint32_t kChunkB = 32 * 16;  // one chunk row of the warp
  constexpr uint32_t kStageB = sizeof(LaneStage);
  // this lane's chunk-0 slot of stage 0; its mask slot of a stage is mdelta on
  const uint32_t ring0 = smem_u32(&ring.s[0].c[0][lane]);
  const uint32_t ring_last = ring0 + (RING - 1) * kStageB;
  const uint32_t mdelta = 4 * kChunkB - 12 * lane;
  auto issue = [&](int it, uint32_t dst) {
    if (!FM_HOT_NOLOAD && S * it + sg < nblk) {
      const float4* p1 = x1b + 8 * S * it;
      const float4* p2 = x2b + 8 * S * it;
      cp_async16(dst, p1);
      cp_async16(dst + kChunkB, p1 + 4);
      cp_async16(dst + 2 * kChunkB, p2);
      cp_async16(dst + 3 * kChunkB, p2 + 4);
      cp_async4(dst + mdelta, mwb + ((half0 + kBlkSlots * S * it) >> 5));
    }
    cp_async_commit();
  };
  {  // stale stage bytes must be finite: zero this lane's ring slots once
#pragma unroll
    for (int st = 0; st < RING; ++st)
#pragma unroll
      for (int c = 0; c < 4; ++c) ring.s[st].c[c][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < RING - 1; ++it) issue(it, ring0 + it * kStageB);

  HotAcc<kPrune, kL1, kMom, MOM64> acc;
  acc.zero();
  // cur: the stage read this iteration; prv: the one read last iteration,
  // refilled now (RING - 1 iterations ahead)
  uint32_t cur = ring0, prv = ring_last;
#pragma unroll kUnroll
  for (int it = 0; it < warp_it; ++it) {
    issue(it + RING - 1, prv);
    cp_async_wait<RING - 1>();  // this lane's copies of iteration `it` have landed
    // a block past the item end reads mask 0: nothing counts, nothing is
    // pruned, weights are +0 (its stale ring bytes are finite)
    const int pos = half0 + kBlkSlots * S * it;  // block's first bit, relative to word lo/32
    // this lane's points: slots 2h, 2h+1 (chunk 0) and 2h+8, 2h+9 (chunk 1),
    // i.e. bits 0, 1, 8, 9 of bh (pos is a multiple of 16, so pos % 32 + 2h < 32)
    const uint32_t bh = (S * it + sg < nblk)
                            ? (FM_HOT_NOLOAD ? 0xffffu : lds32(cur + mdelta) >> ((pos & 31) + 2 * h))
                            : 0u;
    uint32_t kept = 0;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float4 x1 = lds128(cur + j * kChunkB);
      const float4 x2 = lds128(cur + (2 + j) * kChunkB);
      kept |= (uint32_t)acc.point(G, x1.x, x1.y, x2.x, x2.y, (bh & (1u << (8 * j))) != 0u, thr) << (8 * j);
      kept |= (uint32_t)acc.point(G, x1.z, x1.w, x2.z, x2.w, (bh & (2u << (8 * j))) != 0u, thr) << (8 * j + 1);
    }
    acc.cnt += __popc(kept);
    const uint32_t cleared = kPrune ? ((bh & 0x303u) & ~kept) << (2 * h) : 0u;
    if (kPrune && cleared) atomicAnd(mwb_w + (pos >> 5), ~(cleared << (pos & 31)));
    prv = cur;
    cur = cur == ring_last ? ring0 : cur + kStageB;
  }
  cp_async_wait<0>();
  if (kL1 && kMom && !MOM64) acc.l1 = acc.l1f;
#ifdef FM_HOT_TRACE
  if (blockDim.x == kGrpWarps * 32) __syncthreads();  // one-shot kernels only (uniform per block)
  if (blockDim.x == kGrpWarps * 32 && threadIdx.x == 0 && blockIdx.x < 16384) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_hot_trace[blockIdx.x][0] = smid;
    g_hot_trace[blockIdx.x][1] = t_start;
    g_hot_trace[blockIdx.x][2] = globaltimer();
  }
#endif

  // ------------------------------------------------------------------ reduce
  // transpose-reduce within the item's lanes; lane g then writes its N/L
  // outputs (consecutive items -> neighbouring SoA stores)
  const bool single = d.single;
  if (kMom && MOM64) {
    constexpr int N = L <= 8 ? 40 : (L == 16 ? 48 : 64);  // 36 moments, count, l1, padding
    double v[N];
#pragma unroll
    for (int k = 0; k < 36; ++k) v[k] = acc.M64[MOM64 ? k : 0];
    v[36] = (double)acc.cnt;
    v[37] = acc.l1;
#pragma unroll
    for (int k = 38; k < N; ++k) v[k] = 0.0;
    group_transpose_reduce<L>(v, lane);
    if (NI == P) {  // staged, row-coalesced stores (see the fp32 path)
      double* stage = reinterpret_cast<double*>(&ring.s[0].c[0][0]);
      const int q = lane / L;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < N / L; ++i) stage[(g * (N / L) + i) * IPW + q] = v[i];
      __syncwarp();
      const int64_t n0 = item - q;
#pragma unroll 1
      for (int t = lane; t < 38 * IPW; t += 32) {
        const int k = t / IPW;
        const int64_t n = n0 + (t % IPW);
        if (n >= item_end) continue;
        const double val = stage[t];
        if (k < 36) out.mom64[(int64_t)k * P + n] = val;
        else if (k == 36) { if (out.n_active) out.n_active[n] = (int32_t)val; }
        else if (kL1 && out.l1) out.l1[n] = val;
      }
    } else if (has_item) {
#pragma unroll
      for (int i = 0; i < N / L; ++i) {
        const int k = g * (N / L) + i;
        if (!single) {
          if (k < 36) static_cast<double*>(part.red)[k * NI + item] = v[i];
          else if (k == 36) static_cast<double*>(part.red)[45 * NI + item] = v[i];
          else if (k == 37) part.l1[item] = v[i];
        } else if (k < 36) {
          out.mom64[k * P + d.n] = v[i];
        } else if (k == 36) {
          if (out.n_active) out.n_active[d.n] = (int32_t)v[i];
        } else if (k == 37) {
          if (kL1 && out.l1) out.l1[d.n] = v[i];
        }
      }
    }
  } else if (kMom) {
    constexpr int N = L == 32 ? 64 : 48;  // 36 moments (hot order), 9 vgrad, count, s0, padding
    float v[N];
#pragma unroll
    for (int k = 0; k < 18; ++k) {
      v[2 * k] = acc.Mp[MOM64 ? 0 : k].x;
      v[2 * k + 1] = acc.Mp[MOM64 ? 0 : k].y;
    }
    // vgrad canonical order v[p*3+q]: 00 01 02 10 11 12 20 21 22
    v[36] = acc.V0.x; v[37] = acc.V0.y; v[38] = acc.V3.x;
    v[39] = acc.V1.x; v[40] = acc.V1.y; v[41] = acc.V3.y;
    v[42] = acc.V2.x; v[43] = acc.V2.y; v[44] = acc.v22;
    v[45] = (float)acc.cnt;
    v[46] = acc.s0f;
#pragma unroll
    for (int k = 47; k < N; ++k) v[k] = 0.f;
    group_transpose_reduce<L>(v, lane);
    const double l1 = kL1 ? group_sum<L>(acc.l1) : 0.0;
    if (NI == P) {
      // every item is a whole pair (item == pair): stage the warp's sums in
      // its idle ring and write each output row as IPW consecutive pairs --
      // a handful of sectors per store instead of one per lane
      float* stage = reinterpret_cast<float*>(&ring.s[0].c[0][0]);
      double* stage_l1 = reinterpret_cast<double*>(stage + N * IPW);
      const int q = lane / L;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < N / L; ++i) stage[(g * (N / L) + i) * IPW + q] = v[i];
      if (g == 0) stage_l1[q] = l1;
      __syncwarp();
      const int64_t n0 = item - q;  // first pair of the warp
#pragma unroll 1
      for (int t = lane; t < 47 * IPW; t += 32) {
        const int vi = t / IPW;
        const int64_t n = n0 + (t % IPW);
        if (n >= item_end) continue;
        const float val = stage[t];
        if (vi < 36) out.mom32[(int64_t)hot_mom_index(vi) * P + n] = val;
        else if (vi < 45) { if (kLin) out.vgrad[(int64_t)(vi - 36) * P + n] = val; }
        else if (vi == 45) { if (out.n_active) out.n_active[n] = (int32_t)val; }
        else out.s0[n] = (double)val;
      }
      if (kL1 && out.l1 && lane < IPW && n0 + lane < item_end) out.l1[n0 + lane] = stage_l1[lane];
    } else if (has_item) {
      // destination of each of the lane's N/L sums: a float column (moment,
      // vgrad or partial), the int count or the fp64 s0
#pragma unroll
      for (int i = 0; i < N / L; ++i) {
        const int vi = g * (N / L) + i;
        const int k = vi < 36 ? hot_mom_index(vi) : vi;
        float* col = nullptr;
        int64_t at = d.n;
        if (!single) {
          col = k < 46 ? static_cast<float*>(part.red) + (int64_t)k * NI : nullptr;
          at = item;
        } else if (k < 36) {
          col = out.mom32 + (int64_t)k * P;
        } else if (k < 45 && kLin) {
          col = out.vgrad + (int64_t)(k - 36) * P;
        }
        if (col) col[at] = v[i];
        if (single && k == 45 && out.n_active) out.n_active[d.n] = (int32_t)v[i];
        if (k == 46) (single ? out.s0 : part.s0)[at] = (double)v[i];
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
        if (MOM64) static_cast<double*>(part.red)[45 * NI + item] = (double)cnt;
        else static_cast<float*>(part.red)[45 * NI + item] = (float)cnt;
        if (kL1) part.l1[item] = l1;
      }
    }
  }
  if (part.ctl) {
    // fused {L1, Z, kept} of the pass (irls_refine's per-pass scalars,
    // ref/epipolar.py:282-291): item sums on the item's lanes, the warp's
    // items in order, then exact integer sums over the warps (totals_add)
    const double il1 = kL1 ? group_sum<L>(acc.l1) : 0.0;
    const double icnt = group_sum<L>((double)acc.cnt);
    double w3[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int q = 0; q < IPW; ++q) {
      const double a = __shfl_sync(0xffffffffu, il1, q * L);
      const double c = __shfl_sync(0xffffffffu, icnt, q * L);
      if (item_base + group * IPW + q < item_end) {
        w3[0] += a;
        w3[1] += c;
        w3[2] += c > 0.0 ? 1.0 : 0.0;
      }
    }
    if (lane == 0)
      totals_add(part.ctl, blockIdx.x * kGrpWarps + (threadIdx.x >> 5), w3[0], w3[1], w3[2]);
  }
#ifdef FM_HOT_TRACE
  if (blockDim.x == kGrpWarps * 32) __syncthreads();
  if (blockDim.x == kGrpWarps * 32 && threadIdx.x == 0 && blockIdx.x < 16384) g_hot_trace[blockIdx.x][3] = globaltimer();
#endif
}

template <unsigned MODE, bool MOM64, int L>
__global__ void __launch_bounds__(kGrpWarps * 32, MOM64 ? FM_HOT_MINB64 : FM_HOT_MINB)
point_pass_hot(const fm_point_store s, const double* __restrict__ ghat, const double thr,
               const int32_t* __restrict__ prev_active, const fm_pass_out out,
               const PartialBufs part) {
  hot_body<MODE, MOM64, L>(s, ghat, thr, prev_active, out, part,
                           (int64_t)blockIdx.x * kGrpWarps + (threadIdx.x >> 5), 0, s.n_items);
}

// Tail-shortened launch: items [0, n1) with L1 lanes per item (the most
// efficient width, in whole waves), the rest with L2 > L1 lanes per item in
// the blocks the scheduler dispatches last -- a tail item then takes
// L1/L2 of the time, so the low-occupancy end of the launch shrinks.
template <unsigned MODE, bool MOM64, int L1, int L2, int RING>
__global__ void __launch_bounds__(kGrpWarps * 32, MOM64 ? FM_HOT_MINB64 : FM_HOT_MINB)
point_pass_hot_mixed(const fm_point_store s, const double* __restrict__ ghat, const double thr,
                     const int32_t* __restrict__ prev_active, const fm_pass_out out,
                     const PartialBufs part, const int64_t nb1, const int64_t n1) {
  if ((int64_t)blockIdx.x < nb1)
    hot_body<MODE, MOM64, L1, RING>(s, ghat, thr, prev_active, out, part,
                              (int64_t)blockIdx.x * kGrpWarps + (threadIdx.x >> 5), 0, s.n_items);
  else
    hot_body<MODE, MOM64, L2, RING>(s, ghat, thr, prev_active, out, part,
                              ((int64_t)blockIdx.x - nb1) * kGrpWarps + (threadIdx.x >> 5), n1, s.n_items);
}

// -------------------------------------------------------------- generic kernel
// API modes: optional z columns, fp64 moments, caller-given residual weights,
// residual output, mask-free sweeps.  Plain scalar code; not on the hot loop.
// COORD: kXY32 = fp32 (x, y), z = 1; kXYZ32 = fp32 (x, y) + z columns;
// kXYZ64 = the caller's fp64 (x, y, z) (x1d / x2d).
enum Coord { kXY32 = 0, kXYZ32 = 1, kXYZ64 = 2 };

template <int COORD, bool F64, unsigned MODE>
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
  if (out.stop && *out.stop) return;  // an earlier stage failed: leave everything alone
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
        double a, bb, c, d, e, f;
        if (COORD == kXYZ64) {
          a = s.x1d[3 * sl], bb = s.x1d[3 * sl + 1], e = s.x1d[3 * sl + 2];
          c = s.x2d[3 * sl], d = s.x2d[3 * sl + 1], f = s.x2d[3 * sl + 2];
        } else {
          a = s.x1[2 * sl], bb = s.x1[2 * sl + 1];
          c = s.x2[2 * sl], d = s.x2[2 * sl + 1];
          e = COORD == kXYZ32 ? (double)s.x1z[sl] : 1.0;
          f = COORD == kXYZ32 ? (double)s.x2z[sl] : 1.0;
        }
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

template <unsigned MODE, bool MOM64, int L1, int L2, int RING>
int launch_hot_mixed(const fm_point_store& s, double thr, const double* ghat,
                     const int32_t* prev_active, const fm_pass_out& out, const PartialBufs& part,
                     cudaStream_t stream, int64_t n1) {
  const size_t smem = kGrpWarps * sizeof(LaneRingT<RING>);
  static bool attr = false;
  if (!attr) {
    FM_CUDA(cudaFuncSetAttribute(point_pass_hot_mixed<MODE, MOM64, L1, L2, RING>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int64_t nb1 = n1 / (kGrpWarps * (32 / L1));
  const int64_t nb2 = ceil_div(ceil_div(s.n_items - n1, 32 / L2), kGrpWarps);
  point_pass_hot_mixed<MODE, MOM64, L1, L2, RING><<<(unsigned)(nb1 + nb2), kGrpWarps * 32, smem, stream>>>(
      s, ghat, thr, prev_active, out, part, nb1, n1);
  FM_LAUNCHED(point_pass_hot_mixed);
  if (s.n_items > s.n_pairs) {
    combine_kernel<MOM64, MODE><<<(unsigned)ceil_div(s.n_pairs, 128), 128, 0, stream>>>(s, out, part,
                                                                                        !MOM64);
    FM_LAUNCHED(combine_kernel);
  }
  return FM_OK;
}

// Lanes per item L in {4, 8, 16}: blocks are one-shot, so the last wave of
// a launch is partially filled.  Score each L by the filled fraction of its
// waves and a per-item reduction cost (log2(L) transpose-reduce levels plus a
// per-iteration cost for blocks an item leaves idle in its last iteration).
template <unsigned MODE, bool MOM64>
int launch_hot(const fm_point_store& s, double thr, const double* ghat, const int32_t* prev_active,
               const fm_pass_out& out, const PartialBufs& part, cudaStream_t stream) {
  int bps[3] = {1, 1, 1};
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 4>(&bps[0])) return rc;
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 8>(&bps[1])) return rc;
  if (int rc = hot_blocks_per_sm<MODE, MOM64, 16>(&bps[2])) return rc;
  const double mean_blk = s.n_items ? (double)s.n_slots / kBlkSlots / (double)s.n_items : 0.0;
  const int Ls[3] = {4, 8, 16};
  double best = -1.0;
  int pick = 4;
  for (int k = 0; k < 3; ++k) {
    const int L = Ls[k];
    const double S = L / 4;
    const double blocks = std::ceil((double)s.n_items / (32.0 / L) / kGrpWarps);
    const double resident = (double)bps[k] * sm_count();
    const double waves = blocks / resident;
    const double fill = waves / std::ceil(waves);
    // per-item work in iterations (rounded up to S blocks) + reduction (~4 iterations per level)
    const double iters = std::ceil(std::max(mean_blk, 1.0) / S);
    const double useful = std::max(mean_blk, 1.0) / S;
    const double cost = iters + 1.5 * k + 1.0;
    const double score = fill * useful / cost;
    if (score > best * 1.02) {
      best = score;
      pick = L;
    }
  }
  // Whole waves of L = 4 items, the rest of the launch at L = 8 or 16 (see
  // point_pass_hot_mixed) when that rest is under one wave.
  {
    const int64_t G4 = (int64_t)bps[0] * sm_count() * kGrpWarps * 8;  // items per L=4 wave
    const int64_t n1 = (s.n_items / G4) * G4;
    const char* env_mix = getenv("FM_HOT_MIX");
    const bool mix = env_mix ? atoi(env_mix) != 0 : true;
    // (moment passes only: the light L1 pass runs faster with one width)
    constexpr bool kMomPass = (MODE & FM_PASS_MOMENTS) && (MODE & FM_PASS_IRLS);
    if (kMomPass && mix && !getenv("FM_HOT_L") && n1 > 0 &&
        s.n_items > n1 && mean_blk >= 8)
    {
      // Short launches (at most two L = 4 waves; C2: one) run faster with 3
      // ring stages per lane (less prologue per item, more L1 beside the
      // smaller shared-memory ring) and the remainder at L = 8; long ones
      // with 4 stages and the remainder at L = 16.  Measured (ncu medians,
      // C2 / C4 / C5): 5 stages + L = 16 47.5 / 350.5 / 3156 us; 4 + 16
      // 46.6 / 348.0 / 3152; 3 + 16 46.0 / 350.8 / 3183; 3 + 8 44.8 at C2;
      // 4 + 8 348.3 / 3133 against 4 + 16 347.1 / 3130 on the same box.
      const char* env_r = getenv("FM_HOT_SHORT");  // tuning override: 1 short form, 0 long form
      const bool short_launch = env_r ? atoi(env_r) != 0 : n1 / G4 <= 2;
      if (short_launch)
        return launch_hot_mixed<MODE, MOM64, 4, 8, FM_SHORT_RING>(s, thr, ghat, prev_active, out, part, stream, n1);
      return launch_hot_mixed<MODE, MOM64, 4, 16, 4>(s, thr, ghat, prev_active, out, part, stream, n1);
    }
  }
  if (const char* env = getenv("FM_HOT_L")) pick = atoi(env);  // tuning override
  if (pick == 32) return launch_hot_l<MODE, MOM64, 32>(s, thr, ghat, prev_active, out, part, stream);
  if (pick == 16) return launch_hot_l<MODE, MOM64, 16>(s, thr, ghat, prev_active, out, part, stream);
  if (pick == 8) return launch_hot_l<MODE, MOM64, 8>(s, thr, ghat, prev_active, out, part, stream);
  return launch_hot_l<MODE, MOM64, 4>(s, thr, ghat, prev_active, out, part, stream);
}

template <int COORD, bool F64, unsigned MODE>
int launch_generic(const fm_point_store& s, double thr, const double* ghat, const double* res_in,
                   const int32_t* prev_active, const fm_pass_out& out, const PartialBufs& part,
                   cudaStream_t stream) {
  const int64_t blocks = ceil_div(s.n_items, kWarpsPerBlock);
  point_pass_generic<COORD, F64, MODE><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, stream>>>(
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

template <int COORD, bool F64>
int dispatch_generic(unsigned mode, const fm_point_store& s, double thr, const double* ghat,
                     const double* res_in, const int32_t* prev_active, const fm_pass_out& out,
                     const PartialBufs& part, cudaStream_t stream) {
#define FM_CASE(M) \
  if (mode == (M)) return launch_generic<COORD, F64, (M)>(s, thr, ghat, res_in, prev_active, out, part, stream);
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

#ifdef FM_HOT_TRACE
int fm_debug_hot_trace(void* host_out) {
  FM_CUDA(cudaMemcpyFromSymbol(host_out, g_hot_trace, sizeof(g_hot_trace)));
  return FM_OK;
}
#endif

size_t fm_point_pass_scratch_bytes(const fm_point_store* store) {
  if (!store) return 0;
  const size_t ni = (size_t)store->n_items;
  return scratch_round(sizeof(unsigned)) + scratch_round(sizeof(TotCtl)) +
         scratch_round(ni * kNumRed * sizeof(double)) +
         2 * scratch_round(ni * sizeof(double)) + scratch_round(ni * 4 * sizeof(int32_t)) +
         scratch_round((3 * ni + 192) * sizeof(double)) + 256;
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
  const bool d64 = s.x1d != nullptr;
  FM_REQUIRE(d64 == (s.x2d != nullptr), "x1d and x2d must both be set or both NULL");
  FM_REQUIRE((d64 || (s.x1 && s.x2)) && s.active && s.pair_off && s.pair_len && s.pair_item_off &&
                 s.item_pair,
             "incomplete point store");
  FM_REQUIRE(d64 || (((uintptr_t)s.x1 % 16) == 0 && ((uintptr_t)s.x2 % 16) == 0),
             "coordinate columns must be 16-byte aligned");
  const bool homog = s.x1z != nullptr;
  FM_REQUIRE(homog == (s.x2z != nullptr), "x1z and x2z must both be set or both NULL");
  const bool f64 = (mode & FM_PASS_F64) != 0;
  const unsigned m = mode & ~FM_PASS_F64;
  FM_REQUIRE(!d64 || f64 || !(m & FM_PASS_MOMENTS), "fp64-coordinate stores need FM_PASS_F64 moments");
  const bool need_r = m & (FM_PASS_PRUNE | FM_PASS_L1 | FM_PASS_IRLS | FM_PASS_RES_OUT);
  FM_REQUIRE(!need_r || ghat, "mode 0x%x needs ghat", mode);
  FM_REQUIRE(!(m & FM_PASS_RES_IN) || res_in, "FM_PASS_RES_IN needs res_in");
  FM_REQUIRE(!(m & FM_PASS_RES_OUT) || out->residual, "FM_PASS_RES_OUT needs out->residual");
  FM_REQUIRE(!(m & FM_PASS_SKIP_DROPPED) || prev_active, "SKIP_DROPPED needs prev_active");
  if (m & FM_PASS_MOMENTS) {
    FM_REQUIRE(f64 ? out->mom64 != nullptr : out->mom32 != nullptr, "moment output missing");
    if ((m & FM_PASS_IRLS) && !f64) FM_REQUIRE(out->vgrad && out->s0, "IRLS pass needs vgrad/s0");
  }
  PartialBufs part{nullptr, nullptr, nullptr, 0, nullptr, nullptr, nullptr};
  cudaStream_t st = as_stream(stream);
  fm_point_store s2 = s;  // with item descriptors
  double* tot_part = nullptr;
  size_t tot_bytes = 0;
  {
    Scratch sc(scratch, scratch_bytes);
    // at fixed offsets always: a reserved word, then the fused-totals
    // accumulators -- zero when the scratch is first used (the header asks
    // for zeroed scratch), re-armed by totals_finalize_kernel after each use
    sc.take<unsigned>(1);
    TotCtl* sctl = sc.take<TotCtl>(1);
    if (out->totals) {
      tot_bytes = (3 * (size_t)s.n_items + 192) * sizeof(double);
      tot_part = sc.take<double>(3 * (size_t)s.n_items + 192);
      if (s.n_items == s.n_pairs && !getenv("FM_HOT_NOTOT")) {
        part.ctl = sctl;
        part.totals = out->totals;
      }
    }
    if (s.n_items > s.n_pairs) {
      part.red = sc.take<double>((size_t)s.n_items * kNumRed);
      part.s0 = sc.take<double>((size_t)s.n_items);
      part.l1 = sc.take<double>((size_t)s.n_items);
      part.cap = s.n_items;
    }
    if (!s.item_desc) {
      s2.item_desc = sc.take<int32_t>((size_t)s.n_items * 4);
      if (int rc = fm_point_store_describe(&s2, stream)) return rc;
    }
    FM_REQUIRE((sc.used == 0 || scratch) && sc.ok(), "point-pass scratch too small (%zu < %zu)",
               scratch_bytes, sc.used);
  }
  int rc = FM_OK;
  bool fused = false;  // totals computed inside the hot kernel
  bool handled = false;
  if (d64) {
    rc = dispatch_generic<kXYZ64, true>(m, s2, threshold, ghat, res_in, prev_active, *out, part, st);
    handled = true;
  } else if (!homog && s.slot_align >= kBlkSlots && s.slot_align % kBlkSlots == 0) {
    // fp64 moments are the exact default; fp32 (FFMA2 + shifted model) only for IRLS moments
    const bool hot_f64 = f64 || !(m & FM_PASS_MOMENTS);
    if (hot_f64 || (m & FM_PASS_IRLS)) {
      rc = dispatch_hot(m, hot_f64, s2, threshold, ghat, prev_active, *out, part, st, &handled);
      fused = handled && part.ctl != nullptr;
    }
  }
  if (!handled) {
    PartialBufs gp = part;
    gp.totals = nullptr;
    if (homog)
      rc = f64 ? dispatch_generic<kXYZ32, true>(m, s, threshold, ghat, res_in, prev_active, *out, gp, st)
               : dispatch_generic<kXYZ32, false>(m, s, threshold, ghat, res_in, prev_active, *out, gp, st);
    else
      rc = f64 ? dispatch_generic<kXY32, true>(m, s, threshold, ghat, res_in, prev_active, *out, gp, st)
               : dispatch_generic<kXY32, false>(m, s, threshold, ghat, res_in, prev_active, *out, gp, st);
  }
  if (!rc && fused && part.ctl) return launch_totals_finalize(part.ctl, out->totals, st);
  if (rc || !out->totals || fused) return rc;
  // tuning knob FM_HOT_NOTOT: 1 = totals by the separate fm_pass_totals
  // kernel, 2 = no totals at all (the pass alone)
  if (getenv("FM_HOT_NOTOT") && atoi(getenv("FM_HOT_NOTOT")) == 2) return rc;
  // generic kernels / pairs split over several items: a separate reduction
  FM_REQUIRE(out->n_active, "totals need out->n_active");
  return fm_pass_totals((m & FM_PASS_L1) ? out->l1 : nullptr, out->n_active, s.n_pairs, out->totals,
                        tot_part, tot_bytes, stream);
}

}  // extern "C"
