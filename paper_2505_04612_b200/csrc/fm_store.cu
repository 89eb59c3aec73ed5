// Point-pair store construction on the device and the per-pass totals.
//
// fm_store_build turns the caller's point arrays -- every EpipolarPair's x1,
// x2 and active mask (ref/epipolar.py:19-36), concatenated in caller pair
// order -- into the SoA store of fm_point_pass: pairs in stable (i, j) order
// (the caller's order kept as a rank permutation), each pair starting on a
// 16-slot boundary, fp32 (x, y) columns (or the caller's fp64 (x, y, z) for
// API stores), a 1-bit active mask.  The host computes only the O(pairs)
// layout (sort by (i, j), slot offsets); every O(points) step -- the scatter,
// the fp64 -> fp32 conversion, the non-finite sanitising, the mask packing --
// runs here, one warp per caller pair.
//
// fm_store_gather_mask / fm_store_gather_slots map slot-ordered results back
// to caller point order (the in-place mask write-back of ref/epipolar.py:283,
// the per-point residuals of current_residuals ref/epipolar.py:251-255), and
// fm_store_scatter_slots maps caller-ordered values to slots (the residuals
// argument of precompute_weights, ref/epipolar.py:46-59).
//
// fm_pass_totals reduces a pass's per-pair L1 and active counts to the three
// scalars irls_refine needs per pass (ref/epipolar.py:282-291: kept pairs,
// Z, and the L1 sum of epipolar_loss("l1") :156-160) in one launch, in a
// fixed order (bitwise reproducible).
#include "fm_common.cuh"

namespace fm {

namespace {

__device__ __forceinline__ bool finite3(const double* p, int dim) {
  bool ok = isfinite(p[0]) && isfinite(p[1]);
  if (dim == 3) ok = ok && isfinite(p[2]);
  return ok;
}

// One warp per caller pair k: its points [cs[k], cs[k+1]) go to slots
// [pair_off[rank[k]], ...).  32 points per iteration; the warp's active bits
// form one 32-bit ballot that lands in at most two mask words (atomicOr:
// pair starts are 16-slot aligned, so two pairs can share a word).
__global__ void store_build_kernel(fm_point_store s, const double* __restrict__ x1,
                                   const double* __restrict__ x2, int dim,
                                   const uint8_t* __restrict__ act_in,
                                   const int64_t* __restrict__ cs, const int64_t* __restrict__ rank,
                                   int64_t P, int sanitize) {
  const int lane = threadIdx.x & 31;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= P) return;
  const int64_t src = cs[k], len = cs[k + 1] - cs[k];
  const int64_t dst = s.pair_off[rank[k]];
  float2* c1 = reinterpret_cast<float2*>(const_cast<float*>(s.x1));
  float2* c2 = reinterpret_cast<float2*>(const_cast<float*>(s.x2));
  double* d1 = const_cast<double*>(s.x1d);
  double* d2 = const_cast<double*>(s.x2d);
  float* z1 = const_cast<float*>(s.x1z);
  float* z2 = const_cast<float*>(s.x2z);
  for (int64_t b = 0; b < len; b += 32) {
    const int64_t m = b + lane;
    bool on = false;
    if (m < len) {
      const double* p1 = x1 + (src + m) * dim;
      const double* p2 = x2 + (src + m) * dim;
      on = act_in ? act_in[src + m] != 0 : true;
      double a[3] = {p1[0], p1[1], dim == 3 ? p1[2] : 1.0};
      double c[3] = {p2[0], p2[1], dim == 3 ? p2[2] : 1.0};
      if (sanitize && !(finite3(p1, dim) && finite3(p2, dim))) {
        // a non-finite residual fails the first prune (ref/epipolar.py:283)
        a[0] = a[1] = c[0] = c[1] = 0.0;
        a[2] = c[2] = 1.0;
        on = false;
      }
      const int64_t sl = dst + m;
      if (d1) {
        for (int q = 0; q < 3; ++q) {
          d1[3 * sl + q] = a[q];
          d2[3 * sl + q] = c[q];
        }
      } else {
        c1[sl] = make_float2((float)a[0], (float)a[1]);
        c2[sl] = make_float2((float)c[0], (float)c[1]);
        if (z1) {
          z1[sl] = (float)a[2];
          z2[sl] = (float)c[2];
        }
      }
    }
    const unsigned bits = __ballot_sync(0xffffffffu, on);
    if (lane == 0 && bits) {
      const int64_t s0 = dst + b;  // slot of bit 0
      const int sh = (int)(s0 & 31);
      atomicOr(&s.active[s0 >> 5], bits << sh);
      if (sh) atomicOr(&s.active[(s0 >> 5) + 1], bits >> (32 - sh));
    }
  }
}

// slot-ordered -> caller point order (warp per caller pair)
template <typename F>
__global__ void caller_gather_kernel(const int64_t* __restrict__ pair_off,
                                     const int64_t* __restrict__ cs,
                                     const int64_t* __restrict__ rank, int64_t P, F f) {
  const int lane = threadIdx.x & 31;
  const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= P) return;
  const int64_t src = cs[k], len = cs[k + 1] - cs[k];
  const int64_t dst = pair_off[rank[k]];
  for (int64_t m = lane; m < len; m += 32) f(src + m, dst + m);
}

// fixed-order totals: block b sums pairs [b*chunk, (b+1)*chunk) with a
// fixed tree; the last block (ticket) adds the block partials in order
constexpr int kTotBlocks = 64;
constexpr int kTotThreads = 256;

__global__ void pass_totals_kernel(const double* __restrict__ l1, const int32_t* __restrict__ cnt,
                                   int64_t P, double* __restrict__ part, unsigned* ticket,
                                   double* __restrict__ out) {
  __shared__ double s_l1[kTotThreads];
  __shared__ long long s_z[kTotThreads], s_k[kTotThreads];
  __shared__ bool last;
  const int64_t per = (P + kTotBlocks - 1) / kTotBlocks;
  const int64_t lo = blockIdx.x * per, hi = min(P, lo + per);
  double a = 0.0;
  long long z = 0, kp = 0;
  for (int64_t n = lo + threadIdx.x; n < hi; n += kTotThreads) {
    if (l1) a += l1[n];
    const int c = cnt[n];
    z += c;
    kp += c > 0;
  }
  s_l1[threadIdx.x] = a;
  s_z[threadIdx.x] = z;
  s_k[threadIdx.x] = kp;
  __syncthreads();
  for (int st = kTotThreads / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      s_l1[threadIdx.x] += s_l1[threadIdx.x + st];
      s_z[threadIdx.x] += s_z[threadIdx.x + st];
      s_k[threadIdx.x] += s_k[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = s_l1[0];
    part[3 * blockIdx.x + 1] = (double)s_z[0];
    part[3 * blockIdx.x + 2] = (double)s_k[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < (int)gridDim.x; ++b)
      for (int q = 0; q < 3; ++q) t[q] += part[3 * b + q];
    for (int q = 0; q < 3; ++q) out[q] = t[q];
  }
}

int check_layout(const fm_point_store* s) {
  FM_REQUIRE(s && s->pair_off && s->active, "incomplete store");
  FM_REQUIRE((s->x1d != nullptr) == (s->x2d != nullptr), "x1d and x2d must both be set or both NULL");
  FM_REQUIRE(s->x1d || (s->x1 && s->x2), "store needs fp32 or fp64 coordinate columns");
  FM_REQUIRE((s->x1z != nullptr) == (s->x2z != nullptr), "x1z and x2z must both be set or both NULL");
  return FM_OK;
}

unsigned warps_blocks(int64_t warps) { return (unsigned)ceil_div(warps * 32, 256); }

}  // namespace

}  // namespace fm

using namespace fm;

extern "C" {

int fm_store_build(const fm_point_store* store, const double* x1, const double* x2, int32_t dim,
                   const uint8_t* active_in, const int64_t* caller_start,
                   const int64_t* caller_rank, int32_t sanitize, void* stream) {
  if (int rc = check_layout(store)) return rc;
  FM_REQUIRE(dim == 2 || dim == 3, "dim must be 2 or 3");
  FM_REQUIRE(caller_start && caller_rank, "caller_start / caller_rank missing");
  cudaStream_t st = as_stream(stream);
  const fm_point_store& s = *store;
  FM_CUDA(cudaMemsetAsync(s.active, 0, (size_t)(s.n_slots / 32) * sizeof(uint32_t), st));
  if (s.x1d) {
    FM_CUDA(cudaMemsetAsync(const_cast<double*>(s.x1d), 0, (size_t)s.n_slots * 3 * sizeof(double), st));
    FM_CUDA(cudaMemsetAsync(const_cast<double*>(s.x2d), 0, (size_t)s.n_slots * 3 * sizeof(double), st));
  } else {
    FM_CUDA(cudaMemsetAsync(const_cast<float*>(s.x1), 0, (size_t)s.n_slots * 2 * sizeof(float), st));
    FM_CUDA(cudaMemsetAsync(const_cast<float*>(s.x2), 0, (size_t)s.n_slots * 2 * sizeof(float), st));
    if (s.x1z) {
      FM_CUDA(cudaMemsetAsync(const_cast<float*>(s.x1z), 0, (size_t)s.n_slots * sizeof(float), st));
      FM_CUDA(cudaMemsetAsync(const_cast<float*>(s.x2z), 0, (size_t)s.n_slots * sizeof(float), st));
    }
  }
  if (s.n_pairs == 0) return FM_OK;
  FM_REQUIRE(x1 && x2, "null point arrays");
  store_build_kernel<<<warps_blocks(s.n_pairs), 256, 0, st>>>(s, x1, x2, dim, active_in, caller_start,
                                                              caller_rank, s.n_pairs, sanitize);
  FM_LAUNCHED(store_build_kernel);
  return FM_OK;
}

int fm_store_gather_mask(const fm_point_store* store, const int64_t* caller_start,
                         const int64_t* caller_rank, uint8_t* out, void* stream) {
  if (int rc = check_layout(store)) return rc;
  if (store->n_pairs == 0) return FM_OK;
  const uint32_t* act = store->active;
  caller_gather_kernel<<<warps_blocks(store->n_pairs), 256, 0, as_stream(stream)>>>(
      store->pair_off, caller_start, caller_rank, store->n_pairs,
      [=] __device__(int64_t z, int64_t sl) { out[z] = (act[sl >> 5] >> (sl & 31)) & 1u; });
  FM_LAUNCHED(caller_gather_kernel);
  return FM_OK;
}

int fm_store_gather_slots(const fm_point_store* store, const int64_t* caller_start,
                          const int64_t* caller_rank, const double* slot_values, double* out,
                          void* stream) {
  if (int rc = check_layout(store)) return rc;
  if (store->n_pairs == 0) return FM_OK;
  caller_gather_kernel<<<warps_blocks(store->n_pairs), 256, 0, as_stream(stream)>>>(
      store->pair_off, caller_start, caller_rank, store->n_pairs,
      [=] __device__(int64_t z, int64_t sl) { out[z] = slot_values[sl]; });
  FM_LAUNCHED(caller_gather_kernel);
  return FM_OK;
}

int fm_store_scatter_slots(const fm_point_store* store, const int64_t* caller_start,
                           const int64_t* caller_rank, const double* caller_values,
                           double* slot_out, void* stream) {
  if (int rc = check_layout(store)) return rc;
  if (store->n_pairs == 0) return FM_OK;
  caller_gather_kernel<<<warps_blocks(store->n_pairs), 256, 0, as_stream(stream)>>>(
      store->pair_off, caller_start, caller_rank, store->n_pairs,
      [=] __device__(int64_t z, int64_t sl) { slot_out[sl] = caller_values[z]; });
  FM_LAUNCHED(caller_gather_kernel);
  return FM_OK;
}

size_t fm_pass_totals_scratch_bytes(void) {
  return scratch_round(3 * kTotBlocks * sizeof(double)) + scratch_round(sizeof(unsigned)) + 256;
}

int fm_pass_totals(const double* l1, const int32_t* n_active, int64_t n_pairs, double* out3,
                   void* scratch, size_t scratch_bytes, void* stream) {
  FM_REQUIRE(n_active && out3, "fm_pass_totals needs n_active and out3");
  Scratch sc(scratch, scratch_bytes);
  double* part = sc.take<double>(3 * kTotBlocks);
  unsigned* ticket = sc.take<unsigned>(1);
  FM_REQUIRE(scratch && sc.ok(), "fm_pass_totals scratch too small");
  FM_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned), as_stream(stream)));
  pass_totals_kernel<<<kTotBlocks, kTotThreads, 0, as_stream(stream)>>>(l1, n_active, n_pairs, part,
                                                                        ticket, out3);
  FM_LAUNCHED(pass_totals_kernel);
  return FM_OK;
}

}  // extern "C"
