/*
 * fastmap_b200.h -- C ABI of the B200-native FastMap hot path.
 *
 * This is the drop-in boundary for the two gradient-descent stages of the
 * FastMap reference package (/root/reference/pkg/src/fastmap):
 *
 *   epipolar adjustment   ref/epipolar.py:46-319   (precompute_weights,
 *                          current_residuals, epipolar_loss,
 *                          quadratic_loss_and_grad, irls_refine)
 *   global translation    ref/translation.py:112-186 (translation_loss_and_grad,
 *                          align_centers, per_node_residuals, canonicalize,
 *                          multi_init_align)
 *   optimizer / 6D rot    ref/optim.py:11-110       (Adam, rot6d_to_matrix,
 *                          rot6d_jacobian), ref/model.py:112-116 project_to_so3
 *
 * Conventions
 *   - Every array argument is a DEVICE pointer unless the name says host_.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as void*,
 *     NULL = legacy default stream).  No call synchronises the device except
 *     where documented (the *_create helpers).
 *   - Return value is an fm_status.  On failure fm_last_error() returns a
 *     thread-local message.  Asynchronous numerical errors (non-finite loss /
 *     gradient, degenerate 6D rotations) are reported through a device int32
 *     `flag` word which holds the FIRST fm_status code raised; the host maps it
 *     to the same Python exception the reference raises.
 *   - fp64 parameters, fp32 point coordinates.  The packed parameter vector
 *     has the reference layout [rot6d (n x 6) | centers (n x 3) | log_focal (C)]
 *     (ref/epipolar.py:95-106).
 *   - No torch types: plain pointers and sizes only.
 */
#ifndef FASTMAP_B200_H
#define FASTMAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FM_ABI_VERSION 6

typedef enum fm_status {
  FM_OK = 0,
  FM_ERR_INVALID = 1,           /* bad arguments              -> ValueError            */
  FM_ERR_CUDA = 2,              /* CUDA runtime failure       -> RuntimeError          */
  FM_ERR_NONFINITE_LOSS = 3,    /* ref/epipolar.py:306-307    -> FloatingPointError    */
  FM_ERR_NONFINITE_GRAD = 4,    /* ref/optim.py:28-29         -> FloatingPointError    */
  FM_ERR_ROT6D_ZERO = 5,        /* ref/optim.py:50-51         -> ValueError            */
  FM_ERR_ROT6D_COLLINEAR = 6,   /* ref/optim.py:55-56         -> ValueError            */
  FM_ERR_NO_ACTIVE = 7,         /* ref/epipolar.py:147-148    -> ValueError            */
  FM_ERR_ALL_PRUNED = 8,        /* ref/epipolar.py:289-290    -> ValueError            */
  FM_ERR_NONFINITE_TRANSLATION = 9, /* ref/translation.py:149-150 -> FloatingPointError */
  FM_ERR_NONFINITE_ROTATION = 10 /* ref/rotation.py:218-219    -> FloatingPointError   */
} fm_status;

/* ------------------------------------------------------------------------ */
/* library                                                                  */
/* ------------------------------------------------------------------------ */

int fm_abi_version(void);
const char* fm_last_error(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int fm_device_count(void);

/* ------------------------------------------------------------------------ */
/* point-pair store (the per-point data of all EpipolarPair objects)         */
/* ------------------------------------------------------------------------ */
/*
 * Structure of arrays (one (x, y) column per image side, 16 B per point pair),
 * image pairs sorted by (img_i, img_j) (the order of ref/tracks.py:104).  Pair n owns slots [pair_off[n], pair_off[n]+pair_len[n]);
 * pair_off[n] is a multiple of slot_align (>= 4, a power of two) so every
 * 128-bit load belongs to one pair; slot_align >= 16 selects the hot kernel,
 * which moves whole 16-slot blocks without bounds checks.  Padding slots hold
 * zeros and a cleared active bit.  n_slots is a multiple of
 * 128.  The per-point data replaces EpipolarPair.x1/x2/active
 * (ref/epipolar.py:19-36); `terms` is never materialised.
 *
 * A pass is split into work items of at most `chunk` slots (multiple of 128);
 * item k belongs to pair item_pair[k]; pair n owns items
 * [pair_item_off[n], pair_item_off[n+1]).
 */
typedef struct fm_point_store {
  int64_t n_pairs;
  int64_t n_slots;
  int64_t n_items;
  int64_t chunk;
  const int64_t* pair_off;      /* [n_pairs+1] */
  const int32_t* pair_len;      /* [n_pairs]   */
  const int32_t* pair_item_off; /* [n_pairs+1] */
  const int32_t* item_pair;     /* [n_items]   */
  const float* x1;              /* [n_slots][2] image-i normalized (x, y), fp32 */
  const float* x2;              /* [n_slots][2] image-j normalized (x, y), fp32 */
  const float* x1z;             /* [n_slots] or NULL => homogeneous z == 1 (pipeline case) */
  const float* x2z;
  uint32_t* active;             /* [n_slots/32] bit s%32 of word s/32 = slot s active */
  /* [n_items][4] int32 work-item descriptors {slot lo (low, high 32 bits),
   * points, pair | single-item-pair << 31}, filled by fm_point_store_describe;
   * NULL = derived into scratch on every pass. */
  int32_t* item_desc;
  int64_t slot_align;           /* alignment of pair_off (slots): 4 or a multiple of 16 */
  /* [n_slots][3] fp64 (x, y, z) columns or NULL.  When set, every pass reads
   * the caller's fp64 coordinates (the API functions precompute_weights,
   * current_residuals and epipolar_loss take fp64 arrays,
   * ref/epipolar.py:46-59, :141-160, :251-255) through the generic kernel;
   * x1/x2/x1z/x2z may then be NULL.  Moment passes need FM_PASS_F64. */
  const double* x1d;
  const double* x2d;
} fm_point_store;

/*
 * Build the store on the device from the caller's point arrays: x1, x2 are
 * [Z][dim] fp64 (dim 2: z == 1, or 3), every EpipolarPair's x1 / x2
 * (ref/epipolar.py:19-36) concatenated in CALLER pair order; active_in [Z]
 * uint8 (NULL = all active); caller_start [P+1] the caller-order point
 * offsets; caller_rank [P] the stored (i, j)-sorted position of caller pair
 * k.  The store's layout fields (pair_off, n_slots, ...) and output columns
 * must be set: fp32 x1/x2 (+ x1z/x2z when z != 1) or fp64 x1d/x2d.  Writes
 * the coordinate columns (padding zeroed) and the packed active bits.
 * sanitize != 0 zeroes non-finite points and clears their bit (a non-finite
 * residual fails the first prune, ref/epipolar.py:283).
 */
int fm_store_build(const fm_point_store* store, const double* x1, const double* x2,
                   int32_t dim, const uint8_t* active_in, const int64_t* caller_start,
                   const int64_t* caller_rank, int32_t sanitize, void* stream);

/* Active bit of every caller point, caller order: out [Z] uint8 (the
 * in-place mask write-back of ref/epipolar.py:283). */
int fm_store_gather_mask(const fm_point_store* store, const int64_t* caller_start,
                         const int64_t* caller_rank, uint8_t* out, void* stream);

/* out[z] = slot_values[slot of caller point z] (per-point pass outputs in
 * caller order, e.g. current_residuals ref/epipolar.py:251-255). */
int fm_store_gather_slots(const fm_point_store* store, const int64_t* caller_start,
                          const int64_t* caller_rank, const double* slot_values,
                          double* out, void* stream);

/* slot_out[slot of caller point z] = caller_values[z] (caller-order inputs,
 * e.g. the residuals argument of precompute_weights ref/epipolar.py:46-59). */
int fm_store_scatter_slots(const fm_point_store* store, const int64_t* caller_start,
                           const int64_t* caller_rank, const double* caller_values,
                           double* slot_out, void* stream);

/*
 * The three scalars irls_refine needs after a pass (ref/epipolar.py:282-291,
 * :156-160): out3 = {sum l1 (l1 may be NULL -> 0), Z = sum n_active,
 * kept = #pairs with n_active > 0}, in one launch and a fixed order.
 */
size_t fm_pass_totals_scratch_bytes(void);
int fm_pass_totals(const double* l1, const int32_t* n_active, int64_t n_pairs, double* out3,
                   void* scratch, size_t scratch_bytes, void* stream);

/* Fill store->item_desc from the pair / item arrays (one small kernel). */
int fm_point_store_describe(const fm_point_store* store, void* stream);

/* Pass mode bits (combine with |). */
#define FM_PASS_PRUNE        1u   /* active &= |r| <= threshold  (ref/epipolar.py:283) */
#define FM_PASS_L1           2u   /* l1[n] = sum |r| over pre-prune active (ref :156-160) */
#define FM_PASS_MOMENTS      4u   /* W moments over post-prune active (ref :46-59)      */
#define FM_PASS_IRLS         8u   /* weights 1/max(|r|,1e-6) from the pass' own residual */
#define FM_PASS_ALL_POINTS  16u   /* ignore the mask (current_residuals, ref :251-255)  */
#define FM_PASS_RES_OUT     32u   /* residual[s] = |r| for every slot                   */
#define FM_PASS_RES_IN      64u   /* weights 1/max(|res_in[s]|,1e-6) (precompute_weights) */
#define FM_PASS_F64        128u   /* fp64 moment accumulation (API precision)           */
#define FM_PASS_SKIP_DROPPED 256u /* skip pairs with prev_active[n] == 0                */

/*
 * Per-pair outputs of a point pass (SoA, index [k * n_pairs + n]).
 * W = sum_m w_m t_m t_m^T with t_m = flatten(x2 x1^T) has Kronecker structure:
 * W[(p,r),(q,s)] = mom[sym(p,q)*6 + sym(r,s)], sym in (00,01,02,11,12,22), so
 * 36 moments describe it exactly.  IRLS passes also emit the linearisation
 * terms vgrad = sum w r0 t and s0 = sum w r0^2 of the shifted quadratic model
 * (see DESIGN.md "shifted quadratic model").
 */
typedef struct fm_pass_out {
  float* mom32;       /* [36][n_pairs] or NULL */
  double* mom64;      /* [36][n_pairs] or NULL (FM_PASS_F64) */
  float* vgrad;       /* [9][n_pairs]  or NULL */
  double* s0;         /* [n_pairs]     or NULL */
  double* l1;         /* [n_pairs]     or NULL */
  int32_t* n_active;  /* [n_pairs]     or NULL; post-prune active count */
  double* residual;   /* [n_slots]     or NULL; FM_PASS_RES_OUT */
  /* [3] or NULL: {sum of l1 (0 without FM_PASS_L1), Z = sum of n_active,
   * kept pairs = #(n_active > 0)} of this pass -- the scalars irls_refine
   * needs per pass (ref/epipolar.py:282-291, :156-160); needs n_active.  The
   * hot kernel (one work item per pair) accumulates them exactly in 64-bit
   * integer sums (L1 as fixed point: order-independent, so reproducible) and
   * a one-warp kernel launched after it as a programmatic dependent launch
   * converts them; other passes use one fixed-order reduction kernel. */
  double* totals;
  /* NULL, or a device error word (ABI 6): when it is non-zero at launch the
   * pass does nothing -- in particular a prune leaves the masks alone.
   * irls_refine enqueues its schedule without host round trips; this keeps
   * the caller's masks at the state of the first error, as the reference
   * stops there (ref/epipolar.py:283-308). */
  const int32_t* stop;
} fm_pass_out;

/* Scratch of fm_point_pass.  It must be ZEROED before its first use (the
 * fused-totals accumulators live at fixed offsets; every pass that uses them
 * leaves them zero again).  One pass at a time per scratch (stream order). */
size_t fm_point_pass_scratch_bytes(const fm_point_store* store);

/*
 * One fused sweep over all point pairs: residual r = x2^T Ghat_n x1 (fp64),
 * optional prune, L1 partials, IRLS-weighted W moments and linearisation
 * terms.  ghat = [9][n_pairs] fp64 (row-major Ghat_n), may be NULL when the
 * mode needs no residual.  res_in = [n_slots] fp64 for FM_PASS_RES_IN.
 * prev_active = [n_pairs] for FM_PASS_SKIP_DROPPED.
 */
int fm_point_pass(const fm_point_store* store, unsigned mode, double threshold,
                  const double* ghat, const double* res_in,
                  const int32_t* prev_active, const fm_pass_out* out,
                  void* scratch, size_t scratch_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* image-pair graph of the epipolar adjustment                               */
/* ------------------------------------------------------------------------ */
/*
 * Pairs in store order.  pair_i/pair_j are DENSE image indices (positions in
 * the sorted image_ids of ref/epipolar.py:271); pair_ci/pair_cj are camera ids
 * (ref/epipolar.py:167-168, not remapped).  Incidence lists make the per-image
 * and per-camera gradient reductions deterministic gathers (no float atomics):
 * entries are (pair << 1) | side, side 0 = the image/camera is the pair's i.
 * Camera lists are cut into chunks of <= 1024 incidences (store.CAM_CHUNK): chunk k covers
 * cam_inc[cam_chunk_lo[k] .. cam_chunk_lo[k+1]) and belongs to camera
 * cam_chunk_cam[k]; camera c owns chunks [cam_chunk_off[c], cam_chunk_off[c+1]).
 */
typedef struct fm_pair_graph {
  int32_t n_images;
  int32_t n_cameras;
  int32_t refine_focal;
  int32_t n_cam_chunks;
  int64_t n_pairs;
  const int32_t* pair_i;
  const int32_t* pair_j;
  const int32_t* pair_ci;
  const int32_t* pair_cj;
  const int32_t* img_off;       /* [n_images+1] */
  const int32_t* img_inc;
  const int32_t* cam_off;       /* [n_cameras+1] */
  const int32_t* cam_inc;
  const int32_t* cam_chunk_lo;  /* [n_cam_chunks+1] */
  const int32_t* cam_chunk_cam; /* [n_cam_chunks]   */
  const int32_t* cam_chunk_off; /* [n_cameras+1]    */
} fm_pair_graph;

/* Quadratic model kinds */
#define FM_QUAD_SHIFTED32 0  /* hot path: mom32 + vgrad + s0 about ghat0           */
#define FM_QUAD_W64       1  /* caller-given dense W, row-major [81][n_pairs]       */
#define FM_QUAD_MOM64     2  /* Kronecker moments in fp64 [36][n_pairs], no shift   */

typedef struct fm_quad_model {
  int32_t kind;
  const float* mom32;
  const float* vgrad;
  const double* s0;
  const double* ghat0;   /* [9][n_pairs] linearisation point */
  const double* w81;
  const double* mom64;
} fm_quad_model;

size_t fm_epi_scratch_bytes(const fm_pair_graph* g);

/* ghat[9][n_pairs] of the current state (ref/epipolar.py:109-138). */
int fm_epi_pair_ghat(const fm_pair_graph* g, const double* params, double* ghat,
                     int32_t* flag, void* scratch, size_t scratch_bytes, void* stream);

/*
 * Loss (2/Z) sum ghat^T W ghat and packed gradient (ref/epipolar.py:172-232).
 * scale = 2/Z.  loss_out: one device double.  grad_out: packed, length
 * 9*n_images + (refine_focal ? n_cameras : 0).
 */
int fm_epi_loss_grad(const fm_pair_graph* g, const fm_quad_model* q,
                     const double* params, double scale, double* loss_out,
                     double* grad_out, int32_t* flag, void* scratch,
                     size_t scratch_bytes, void* stream);

/*
 * n_steps fused Adam steps of the quadratic model (the inner loop of
 * ref/epipolar.py:302-308): per step loss/grad + non-finite checks + Adam
 * (ref/optim.py:24-36) on the packed params; t counts from t0+1.
 * use_graph != 0 captures the step sequence in a CUDA graph (cached per
 * argument set) and replays it.
 */
int fm_epi_adam_steps(const fm_pair_graph* g, const fm_quad_model* q,
                      double* params, double* adam_m, double* adam_v,
                      int64_t t0, int32_t n_steps, double lr, double beta1,
                      double beta2, double eps, double scale, int32_t* flag,
                      int32_t use_graph, void* scratch, size_t scratch_bytes,
                      void* stream);

/*
 * fm_epi_adam_steps with scale = 2/Z read on the device from `totals`, the
 * fused {L1, Z, kept} of the round's prune pass (fm_pass_out.totals), so
 * irls_refine enqueues its whole schedule without a host round trip
 * (ref/epipolar.py:291-308).  Z == 0 (every pair pruned) gives an infinite
 * scale and a non-finite flag; the caller checks kept first.
 */
int fm_epi_adam_steps_z(const fm_pair_graph* g, const fm_quad_model* q,
                        double* params, double* adam_m, double* adam_v,
                        int64_t t0, int32_t n_steps, double lr, double beta1,
                        double beta2, double eps, const double* totals,
                        int32_t* flag, int32_t use_graph, void* scratch,
                        size_t scratch_bytes, void* stream);

/*
 * Sharded form of fm_epi_adam_steps: `g` / `q` hold this rank's
 * contiguous range of image pairs (global image / camera indexing); per step
 * the local packed gradient goes to grad_buf [9N + C] and the finiteness of
 * the local loss terms to grad_buf[9N + C] (0 or NaN), one
 * ncclAllReduce(sum) over `nccl_comm` (an ncclComm_t from fm_nccl_comm_init;
 * NULL = one rank) and the replicated Adam step (ref/optim.py:24-36) with
 * the loss check of ref/epipolar.py:306-307 on every rank.  Every rank passes the same
 * params / adam_m / adam_v values and ends with the same results.  With
 * use_graph the chunk, collective included, is one cached CUDA graph.
 */
int fm_epi_adam_steps_nccl(const fm_pair_graph* g, const fm_quad_model* q,
                           double* params, double* adam_m, double* adam_v,
                           int64_t t0, int32_t n_steps, double lr, double beta1,
                           double beta2, double eps, double scale, int32_t* flag,
                           void* nccl_comm, double* grad_buf, int32_t use_graph,
                           void* scratch, size_t scratch_bytes, void* stream);

/*
 * The sharded step with its all-reduce FUSED into the reduce kernel over
 * peer memory: every rank runs it at the same time on its own
 * shard.  Per step pair_grad, then one kernel whose blocks write their local
 * packed-gradient components to this rank's exchange buffer, publish a step
 * id on their ready flag, wait for the same block of every peer, sum the
 * ranks' components in rank order (the same sum everywhere) and apply Adam
 * (ref/optim.py:24-36) -- no separate collective, no grid barrier.  part[r]
 * / ready[r] are device pointers to rank r's buffers (peer memory mapped
 * with fm_ipc_open_handle, or plain device memory for ranks sharing a GPU);
 * the two pointer arrays themselves live in device memory.  Exchange
 * buffers hold 2 * fm_peer_part_len doubles, flag arrays fm_peer_flag_len
 * u64 (zeroed once); epoch = steps this group completed before the call.
 * At most 8 refined cameras.  A peer that never arrives raises FM_ERR_CUDA
 * after ~1 s of waiting instead of hanging.
 */
typedef struct fm_peer_group {
  int32_t n_ranks;
  int32_t rank;
  double* const* part;
  unsigned long long* const* ready;
  int64_t epoch;
  int32_t max_blocks;  /* cap on the kernel's blocks (0: what is resident); ranks sharing a GPU */
  int32_t system_scope; /* 1: peers on other GPUs (system-scope release/acquire); 0: one GPU */
} fm_peer_group;

size_t fm_peer_part_len(const fm_pair_graph* g);
size_t fm_peer_flag_len(const fm_pair_graph* g);
int fm_epi_adam_steps_peer(const fm_pair_graph* g, const fm_quad_model* q,
                           double* params, double* adam_m, double* adam_v,
                           int64_t t0, int32_t n_steps, double lr, double beta1,
                           double beta2, double eps, double scale, int32_t* flag,
                           const fm_peer_group* group, int32_t use_graph,
                           void* scratch, size_t scratch_bytes, void* stream);

/* This rank's exchange buffers (cudaMalloc, zeroed): *part [2][part_doubles]
 * doubles, *ready [n_flags] u64 -- whole allocations, so they can be shared
 * with fm_ipc_get_handle. */
int fm_peer_buffers_alloc(size_t part_doubles, size_t n_flags, double** part,
                          unsigned long long** ready);
int fm_peer_buffers_free(double* part, unsigned long long* ready);
/* In-place sum of n <= 32 doubles over the ranks of a peer group (the pass
 * scalars of irls_refine, ref/epipolar.py:282-291, in the sharded step):
 * one warp publishes vals into this rank's exchange buffer (2 x n doubles,
 * flag array of 1), waits for every peer and sums in rank order (the same
 * result everywhere).  group->epoch = exchanges completed before this one;
 * *err gets FM_ERR_CUDA if a peer never arrives (bounded wait). */
int fm_peer_sum_f64(double* vals, int32_t n, const fm_peer_group* group, int32_t* err,
                    void* stream);
/* CUDA IPC of exchange buffers between the ranks' processes (64-byte
 * handles, exchanged out of band). */
int fm_ipc_get_handle(const void* dev_ptr, void* handle_out);
int fm_ipc_open_handle(const void* handle, void** dev_ptr_out);
int fm_ipc_close_handle(void* dev_ptr);

/* Drop every CUDA graph cached by fm_epi_adam_steps (use_graph != 0). */
void fm_release_cached_graphs(void);

/* rot6d -> SO(3) (ref/optim.py:39-59); project != 0 additionally applies the
 * polar projection of ref/model.py:112-116.  R_out [n][9] row-major. */
int fm_rot6d_to_matrix(const double* rot6d, int64_t n, int32_t project,
                       double* R_out, int32_t* flag, void* stream);

/* Jacobian of rot6d_to_matrix, [n][9][6] (ref/optim.py:68-110). */
int fm_rot6d_jacobian(const double* rot6d, int64_t n, double* J_out,
                      void* stream);

/* Batched polar projection of arbitrary 3x3 matrices onto SO(3)
 * (ref/model.py:112-116). */
int fm_project_to_so3(const double* M, int64_t n, double* R_out, void* stream);

/* E = [t]x R_j R_i^T, t = -R_j (o_j - o_i)  (ref/epipolar.py:62-70). */
int fm_compose_essential(const double* R_i, const double* R_j,
                         const double* o_i, const double* o_j, int64_t n,
                         double* E_out, void* stream);

/* One Adam step on a flat fp64 vector (ref/optim.py:24-36).  t >= 1. */
int fm_adam_step(double* params, double* adam_m, double* adam_v,
                 const double* grad, int64_t n, int64_t t, double lr,
                 double beta1, double beta2, double eps, int32_t* flag,
                 void* stream);

/* ------------------------------------------------------------------------ */
/* global translation (direction graph)                                      */
/* ------------------------------------------------------------------------ */
/*
 * DirectionGraph (ref/translation.py:104-109) plus a node incidence list
 * node_inc[node_off[v] .. node_off[v+1]) of (edge << 1) | side, side 0 = v is
 * the edge's i.  Per node the list holds the edges where v is j (side 1) by
 * ascending edge id, then the edges where v is i (side 0) by ascending edge
 * id: the order of the reference's np.add.at scatter
 * (ref/translation.py:123-124).  The kernels fold in this order, which makes
 * every loss, gradient and trajectory bitwise the reference's.  Centres of B
 * independent runs are stored node-major [n][B][3] fp64 so one gather serves
 * all runs.
 */
typedef struct fm_dir_graph {
  int32_t n_nodes;
  int64_t n_edges;
  const int32_t* edge_i;
  const int32_t* edge_j;
  const double* dirs;       /* [n_edges][3] unit world directions */
  const int32_t* node_off;  /* [n_nodes+1] */
  const int32_t* node_inc;
} fm_dir_graph;

size_t fm_tr_scratch_bytes(int32_t n_nodes, int64_t n_edges, int32_t n_runs);

/* Mean per-edge L1 direction loss and gradient, per run
 * (ref/translation.py:112-125).  loss_out [B], grad_out [n][B][3]. */
int fm_tr_loss_grad(const fm_dir_graph* g, const double* centers, int32_t n_runs,
                    double* loss_out, double* grad_out, void* scratch,
                    size_t scratch_bytes, void* stream);

/*
 * B independent Adam descents of the L1 direction loss, in lock-step
 * (ref/translation.py:137-152 for each run).  centers [n][B][3] in/out.
 * loss_out[b] = loss evaluated at the last step (before its update), as the
 * reference returns it.  Adam state is fresh (t = 1..steps).
 */
int fm_tr_align(const fm_dir_graph* g, double* centers, int32_t n_runs,
                int32_t steps, double lr, double beta1, double beta2,
                double eps, double* loss_out, int32_t* flag, void* scratch,
                size_t scratch_bytes, void* stream);

/* canonicalize each run in place (ref/translation.py:128-134). */
int fm_tr_canonicalize(double* centers, int32_t n_nodes, int32_t n_runs,
                       void* scratch, size_t scratch_bytes, void* stream);

/* Mean incident-edge L1 residual per node and run, out [n][B]
 * (ref/translation.py:155-166). */
int fm_tr_node_residuals(const fm_dir_graph* g, const double* centers,
                         int32_t n_runs, double* out, void* stream);

/* Multi-init merge (ref/translation.py:178-184): canonicalize every run,
 * per-node argmin of the mean incident residual (ties -> lowest run), gather.
 * centers [n][B][3] is canonicalized in place; merged [n][3]; choice [n]. */
int fm_tr_merge(const fm_dir_graph* g, double* centers, int32_t n_runs,
                double* merged, int32_t* choice, void* scratch,
                size_t scratch_bytes, void* stream);

/* ------------------------------------------------------------------------ */
/* relative-translation sphere search (SURVEY 8f "next" #1)                  */
/* ------------------------------------------------------------------------ */
/*
 * Mean absolute epipolar error of every candidate direction of one image pair
 * (ref/translation.py:52-55, `_mean_epipolar_errors`):
 *   errors[c] = (1/M) sum_m | x2_m^T [d_c]_x R x1_m |
 * x1, x2: [M][3] normalized homogeneous points (fp64), R: [3][3] relative
 * rotation (frame i -> j, row-major), dirs: [C][3] unit candidates.
 */
int fm_sphere_errors(const double* x1, const double* x2, int64_t M, const double* R,
                     const double* dirs, int32_t C, double* errors_out, void* stream);

/*
 * Cheirality counts of a relative pose and its mirrored translation
 * (ref/twoview.py:246-253 `_positive_depth_count` on (R, t) and (R, -t)):
 * each point pair triangulated by the linear (DLT) method -- the right
 * singular vector of the 4x4 system for its smallest singular value -- and
 * counted when in front of both cameras.  counts_out: 2 int32 (t, -t).
 */
int fm_depth_counts(const double* R, const double* t, const double* x1,
                    const double* x2, int64_t M, int32_t* counts_out, void* stream);

/*
 * Batched forms over n_pairs image pairs (pair k owns points
 * [pair_off[k], pair_off[k+1]) of x1 / x2, rotation R + 9k):
 * errors_out [k][C] with candidates dirs + k * dir_stride (dir_stride 0: one
 * lattice for all pairs); counts_out [k][2] over the first
 * min(M_k, max_points) points with translation t + 3k.  n_pairs <= 65535.
 */
int fm_sphere_errors_batch(const double* x1, const double* x2, const int64_t* pair_off,
                           int32_t n_pairs, const double* R, const double* dirs,
                           int64_t dir_stride, int32_t C, double* errors_out, void* stream);
int fm_depth_counts_batch(const double* R, const double* t, const double* x1,
                          const double* x2, const int64_t* pair_off, int32_t n_pairs,
                          int64_t max_points, int32_t* counts_out, void* stream);

/* ------------------------------------------------------------------------ */
/* rotation refinement (SURVEY 8f "next" #3)                                 */
/* ------------------------------------------------------------------------ */
/*
 * Relative-rotation graph over dense node indices: edge e maps frame
 * edge_i[e] to frame edge_j[e] by rel[e] (row-major 3x3); node_inc lists
 * (e << 1) | side per node (side 1: the node is the edge's j), CSR node_off.
 */
typedef struct fm_rot_graph {
  int32_t n_nodes;
  int64_t n_edges;
  const int32_t* edge_i;
  const int32_t* edge_j;
  const double* rel;        /* [n_edges][9] */
  const int32_t* node_off;  /* [n_nodes+1] */
  const int32_t* node_inc;
} fm_rot_graph;

size_t fm_rot_scratch_bytes(int32_t n_nodes, int64_t n_edges);

/* Mean geodesic loss over edges and its gradient w.r.t. the 6D parameters
 * (ref/rotation.py:162-194).  params6 [n][6]; loss_out: one device double;
 * grad_out [n][6]. */
int fm_rot_loss_grad(const fm_rot_graph* g, const double* params6, double* loss_out,
                     double* grad_out, int32_t* flag, void* scratch, size_t scratch_bytes,
                     void* stream);

/*
 * Adam descent of the mean geodesic loss with the reference's best-iterate
 * and early-stopping rules (ref/rotation.py:197-230): up to max_steps steps,
 * stopping after a loss < 1e-12 or a relative change < 1e-9 over 100 steps.
 * params6 [n][6]: in = initial, out = the best iterate; history_out
 * [max_steps] losses; *steps_out (host int) = losses recorded.  Runs on the
 * stream in CUDA-graph chunks and synchronises once per chunk to test the
 * stop condition.
 */
int fm_rot_refine(const fm_rot_graph* g, double* params6, int32_t max_steps, double lr,
                  double beta1, double beta2, double eps, double* history_out,
                  int32_t* steps_out, int32_t* flag, void* scratch, size_t scratch_bytes,
                  void* stream);

/*
 * Distortion candidate scoring (ref/distortion.py:90-126): for every job =
 * one (candidate alpha, image pair) with M >= 8 undistorted, scaled point
 * pairs p1/p2 [n_points][2] fp64 (rows [job_off[k], job_off[k+1])), the
 * robust fundamental-matrix fit of ref/twoview.py:58-104 (LMedS over the
 * reference's 64 seeded 8-point samples when M >= 16: sample_idx +
 * sample_off[k] holds them as [64][8] int32, sample_off[k] = -1 below 16)
 * and _refit_on_inliers (:48-55), then err_sum[k] = sum |x2^T F x1| and
 * n_err[k] = M -- or n_err[k] = 0 when a fit is degenerate (the reference
 * raises DegenerateGeometryError and score_alpha skips the pair).  F_out
 * (nullable) [n_jobs][9]: the fitted, Frobenius-normalised F row-major
 * (NaN when degenerate).  Replaces the per-pair body of score_alpha
 * (ref/distortion.py:107-124) and, with F_out, batches estimate_fundamental
 * for undistorted_fundamentals (ref/focal.py:51-78).
 */
size_t fm_fund_scratch_bytes(int64_t n_points);
int fm_fund_score(int64_t n_jobs, const int64_t* job_off, const double* p1, const double* p2,
                  const int32_t* sample_idx, const int64_t* sample_off, double* err_sum,
                  int32_t* n_err, double* F_out, void* scratch, size_t scratch_bytes,
                  int64_t n_points, void* stream);

/*
 * Robust homography fit (ref/twoview.py:136-201) for every job (same layout
 * as fm_fund_score, M >= 4 points; sample_off[k] = -1 below 12, else the
 * offset of the reference's 64 sequential 4-point samples [64][4] int32).
 * H_out [n_jobs][9]: Frobenius-normalised, positive-trace H row-major, NaN
 * where the reference raises DegenerateGeometryError.  Scratch:
 * fm_fund_scratch_bytes(n_points).  Batches the homography pairs of
 * apply_calibration (ref/focal.py:195-200).
 */
int fm_homog_fit(int64_t n_jobs, const int64_t* job_off, const double* p1, const double* p2,
                 const int32_t* sample_idx, const int64_t* sample_off, double* H_out,
                 void* scratch, size_t scratch_bytes, int64_t n_points, void* stream);

/*
 * Connected components of the keypoint match graph (build_tracks,
 * ref/tracks.py:38-56): n_nodes (image, keypoint) ids, n_edges
 * correspondences u[e] -- v[e].  labels_out[x] = the smallest node id of
 * x's component.  Synchronises the stream once per hook round.
 */
int fm_cc_labels(int32_t n_nodes, int64_t n_edges, const int32_t* u, const int32_t* v,
                 int32_t* labels_out, void* stream);

/*
 * Focal voting (ref/focal.py:43-48, :81-120): votes_out[c] = sum over pairs
 * p of exp((1 - s0/s1) / tau), s the singular values of E = K2^T F_p K1,
 * K = [[f, 0, cx], [0, f, cy], [0, 0, 1]].  F [n_pairs][9] row-major;
 * focal [n_cand][n_pairs][2] (image-i side, image-j side) -- the candidate
 * focal or a known camera's; principal [n_pairs][4] (cx1, cy1, cx2, cy2).
 */
int fm_focal_votes(int32_t n_cand, int32_t n_pairs, const double* F, const double* focal,
                   const double* principal, double tau, double* votes_out, void* stream);

/* ------------------------------------------------------------------------ */
/* multi-GPU: NCCL communicator (SURVEY 8b "a multi-GPU variant of each takes */
/* an ncclComm_t"; libnccl.so.2 is loaded at run time)                        */
/* ------------------------------------------------------------------------ */
#define FM_NCCL_UNIQUE_ID_BYTES 128

/* 1 when libnccl.so.2 could be loaded, else 0. */
int fm_nccl_available(void);
/* ncclGetUniqueId into id_out [FM_NCCL_UNIQUE_ID_BYTES] (rank 0; the ranks
 * exchange it out of band, e.g. a torch.distributed broadcast). */
int fm_nccl_unique_id(void* id_out);
/* ncclCommInitRank on the current CUDA device; *comm_out is an ncclComm_t. */
int fm_nccl_comm_init(void** comm_out, int32_t n_ranks, const void* id, int32_t rank);
int fm_nccl_comm_destroy(void* comm);
/* In-place sum all-reduce of n doubles (the pass scalars of irls_refine,
 * ref/epipolar.py:282-291); comm NULL = one rank (no-op). */
int fm_nccl_allreduce_sum_f64(double* buf, int64_t n, void* comm, void* stream);
/* recv [n_ranks][n] <- every rank's send [n], rank order (the multi-init
 * translation merge, ref/translation.py:181-185). */
int fm_nccl_allgather_f64(const double* send, double* recv, int64_t n, void* comm,
                          void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FASTMAP_B200_H */
