// Multi-GPU plumbing of the sharded hot path: the C ABI's
// ncclComm_t entry points.  NCCL is resolved at run time with dlopen -- the
// libnccl.so.2 torch.distributed already loaded when there is one (same
// library, so one NCCL per process), else the system one -- so the library
// still loads on hosts without NCCL or GPU.  The communicator is our own
// (ncclCommInitRank over a unique id the ranks exchange through any
// torch.distributed backend); every collective is stream-ordered on the
// caller's stream and CUDA-graph capturable.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "fm_common.cuh"

namespace fm {

namespace {

struct NcclApi {
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  bool loaded = false;
};

const NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define FM_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    FM_SYM(get_unique_id, "ncclGetUniqueId");
    FM_SYM(comm_init_rank, "ncclCommInitRank");
    FM_SYM(comm_destroy, "ncclCommDestroy");
    FM_SYM(comm_count, "ncclCommCount");
    FM_SYM(comm_user_rank, "ncclCommUserRank");
    FM_SYM(all_reduce, "ncclAllReduce");
    FM_SYM(all_gather, "ncclAllGather");
    FM_SYM(error_string, "ncclGetErrorString");
#undef FM_SYM
    api.loaded = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.comm_count &&
                 api.comm_user_rank && api.all_reduce && api.all_gather && api.error_string;
  });
  return api.loaded ? &api : nullptr;
}

int nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi* a = nccl_api();
  return set_error(FM_ERR_CUDA, "%s failed: %s", what, a ? a->error_string(r) : "NCCL unavailable");
}

#define FM_NCCL(call, what)                       \
  do {                                            \
    ncclResult_t r__ = (call);                    \
    if (r__ != ncclSuccess) return nccl_fail(r__, what); \
  } while (0)

}  // namespace

int nccl_allreduce_sum_f64(double* buf, size_t n, void* comm, cudaStream_t st) {
  if (!comm || n == 0) return FM_OK;  // one rank: the sum is the input
  const NcclApi* a = nccl_api();
  FM_REQUIRE(a, "NCCL (libnccl.so.2) could not be loaded");
  FM_NCCL(a->all_reduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), st),
          "ncclAllReduce");
  return FM_OK;
}

// Small all-reduce over peer memory (the pass scalars): one warp per rank
// writes its n values into its exchange buffer (step parity), publishes the
// exchange id, waits for every peer's id and sums the ranks' values in rank
// order -- the same result on every rank.  Bounded spins: a missing peer
// sets *err instead of hanging.
template <bool SYS>
__global__ void peer_sum_kernel(double* vals, int n, double* const* part,
                                unsigned long long* const* ready, int n_ranks, int rank,
                                unsigned long long id, int32_t* err) {
  const int lane = threadIdx.x;
  const int parity = (int)(id & 1);
  double* mine = part[rank] + parity * n;
  if (lane < n) mine[lane] = vals[lane];
  __syncwarp();
  if (lane == 0) {
    if (SYS) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(ready[rank]), "l"(id) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(ready[rank]), "l"(id) : "memory");
  }
  if (lane < n_ranks) {
    long long spins = 0;
    for (;;) {
      unsigned long long v;
      if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(ready[lane]) : "memory");
      else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ready[lane]) : "memory");
      if (v >= id) break;
      __nanosleep(64);
      if (++spins > (1ll << 24)) {
        atomicCAS(err, 0, FM_ERR_CUDA);
        break;
      }
    }
  }
  __syncwarp();
  if (lane < n) {
    double t = 0.0;
    for (int r = 0; r < n_ranks; ++r) t += __ldcv(part[r] + parity * n + lane);
    vals[lane] = t;
  }
}

}  // namespace fm

using namespace fm;

extern "C" {

int fm_peer_sum_f64(double* vals, int32_t n, const fm_peer_group* group, int32_t* err, void* stream) {
  FM_REQUIRE(vals && group && group->part && group->ready && err && n >= 1 && n <= 32,
             "bad peer sum arguments");
  FM_REQUIRE(group->n_ranks >= 1 && group->n_ranks <= 32 && group->rank >= 0 &&
                 group->rank < group->n_ranks && group->epoch >= 0,
             "bad peer group");
  const unsigned long long id = (unsigned long long)group->epoch + 1;
  cudaStream_t st = as_stream(stream);
  if (group->system_scope)
    peer_sum_kernel<true><<<1, 32, 0, st>>>(vals, n, group->part, group->ready, group->n_ranks,
                                            group->rank, id, err);
  else
    peer_sum_kernel<false><<<1, 32, 0, st>>>(vals, n, group->part, group->ready, group->n_ranks,
                                             group->rank, id, err);
  FM_LAUNCHED(peer_sum_kernel);
  return FM_OK;
}

int fm_nccl_available(void) { return nccl_api() ? 1 : 0; }

int fm_nccl_unique_id(void* id_out) {
  FM_REQUIRE(id_out, "null id buffer");
  const NcclApi* a = nccl_api();
  FM_REQUIRE(a, "NCCL (libnccl.so.2) could not be loaded");
  static_assert(sizeof(ncclUniqueId) == FM_NCCL_UNIQUE_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  FM_NCCL(a->get_unique_id(&id), "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return FM_OK;
}

int fm_nccl_comm_init(void** comm_out, int32_t n_ranks, const void* id, int32_t rank) {
  FM_REQUIRE(comm_out && id, "null comm / id");
  FM_REQUIRE(n_ranks >= 1 && rank >= 0 && rank < n_ranks, "bad rank %d of %d", rank, n_ranks);
  const NcclApi* a = nccl_api();
  FM_REQUIRE(a, "NCCL (libnccl.so.2) could not be loaded");
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  FM_NCCL(a->comm_init_rank(&c, n_ranks, uid, rank), "ncclCommInitRank");
  *comm_out = c;
  return FM_OK;
}

int fm_nccl_comm_destroy(void* comm) {
  if (!comm) return FM_OK;
  const NcclApi* a = nccl_api();
  FM_REQUIRE(a, "NCCL (libnccl.so.2) could not be loaded");
  FM_NCCL(a->comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  return FM_OK;
}

int fm_nccl_allreduce_sum_f64(double* buf, int64_t n, void* comm, void* stream) {
  FM_REQUIRE(n >= 0 && (buf || n == 0), "bad buffer");
  return nccl_allreduce_sum_f64(buf, (size_t)n, comm, as_stream(stream));
}

int fm_nccl_allgather_f64(const double* send, double* recv, int64_t n, void* comm, void* stream) {
  FM_REQUIRE(n >= 0 && ((send && recv) || n == 0), "bad buffers");
  cudaStream_t st = as_stream(stream);
  if (!comm) {
    if (n && send != recv) FM_CUDA(cudaMemcpyAsync(recv, send, (size_t)n * sizeof(double),
                                                   cudaMemcpyDeviceToDevice, st));
    return FM_OK;
  }
  const NcclApi* a = nccl_api();
  FM_REQUIRE(a, "NCCL (libnccl.so.2) could not be loaded");
  FM_NCCL(a->all_gather(send, recv, (size_t)n, ncclFloat64, static_cast<ncclComm_t>(comm), st),
          "ncclAllGather");
  return FM_OK;
}

int fm_peer_buffers_alloc(size_t part_doubles, size_t n_flags, double** part, unsigned long long** ready) {
  FM_REQUIRE(part && ready, "null output pointers");
  *part = nullptr;
  *ready = nullptr;
  FM_CUDA(cudaMalloc(reinterpret_cast<void**>(part), std::max<size_t>(2 * part_doubles, 1) * sizeof(double)));
  FM_CUDA(cudaMalloc(reinterpret_cast<void**>(ready), std::max<size_t>(n_flags, 1) * sizeof(unsigned long long)));
  FM_CUDA(cudaMemset(*part, 0, std::max<size_t>(2 * part_doubles, 1) * sizeof(double)));
  FM_CUDA(cudaMemset(*ready, 0, std::max<size_t>(n_flags, 1) * sizeof(unsigned long long)));
  return FM_OK;
}

int fm_peer_buffers_free(double* part, unsigned long long* ready) {
  if (part) FM_CUDA(cudaFree(part));
  if (ready) FM_CUDA(cudaFree(ready));
  return FM_OK;
}

int fm_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  FM_REQUIRE(dev_ptr && handle_out, "null pointer");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  FM_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  memcpy(handle_out, &h, sizeof(h));
  return FM_OK;
}

int fm_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  FM_REQUIRE(handle && dev_ptr_out, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  FM_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return FM_OK;
}

int fm_ipc_close_handle(void* dev_ptr) {
  if (dev_ptr) FM_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return FM_OK;
}

}  // extern "C"
