/*
 * o3g.h — C ABI of the B200-native point-to-plane ICP hot path.
 *
 * The operation is Open3D's registration_icp(source, target,
 * max_correspondence_distance, init, TransformationEstimationPointToPlane())
 * (§3.3): iterate { transform the source by T; find each
 * source point's nearest target point within max_correspondence_distance;
 * form the point-to-plane residual r = (T s - q).n and its 6-DoF Jacobian;
 * reduce J^T J and J^T r; take the Gauss-Newton step of
 * Eq. 2; compose } until the fitness / inlier-rmse criteria
 * of SPEC.md:282-290 hold. Conventions are DESIGN.md §3's readings R1-R14.
 *
 * General rules (every entry point):
 *  - Return an o3g_status; never throw, never abort. O3G_OK is 0.
 *  - Point arrays are float32, row-major [n][3] (x,y,z), contiguous.
 *    4x4 transforms are float64 row-major (16 doubles), rigid: R^T R = I and
 *    det R = +1 within 1e-9, bottom row exactly (0,0,0,1).
 *  - Array pointers may be DEVICE pointers (cudaMalloc / torch CUDA tensors,
 *    on the context's device) or HOST pointers (pageable or pinned); the
 *    library asks the driver which. Host arrays are copied to the device
 *    inside the call (this is the "end-to-end" path). Scalars and 4x4
 *    matrices are always host values.
 *  - Ownership: the library never frees, retains or writes caller arrays
 *    except the documented outputs. An o3g_ctx owns all device memory it
 *    allocates; o3g_destroy releases it.
 *  - Streams: work is ordered on the context's stream (cuda_stream; NULL =
 *    the legacy default stream). Host outputs are valid on return: calls
 *    that return host values synchronise that stream.
 *  - Errors: O3G_ERR_INVALID_ARGUMENT for n <= 0 ("empty ->
 *    invalid-argument"), dmax <= 0 or non-finite, NULL required pointers
 *    (point-to-plane needs target normals), non-rigid T
 *    (SPEC.md:80), negative criteria / iterations, non-finite coordinates
 *    or normals ("non-finite"). O3G_ERR_CUDA / _OUT_OF_MEMORY /
 *    _COMM report runtime failures; o3g_last_error() gives the message.
 *  - Zero correspondences are not an error: O3G_OK, fitness
 *    0, rmse 0, info.flags |= O3G_FLAG_NO_CORRESPONDENCES, T_out = last T.
 *  - A singular 6x6 system stops the loop: O3G_OK with info.flags |=
 *    O3G_FLAG_DEGENERATE and T_out = the last T (R6).
 *  - There is no CPU fallback: without a usable sm_100a device every call
 *    that needs one returns O3G_ERR_CUDA.
 */
#ifndef O3G_H
#define O3G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum {
    O3G_OK = 0,
    O3G_ERR_INVALID_ARGUMENT = 1,
    O3G_ERR_DEGENERATE = 2,
    O3G_ERR_CUDA = 3,
    O3G_ERR_OUT_OF_MEMORY = 4,
    O3G_ERR_COMM = 5,
    O3G_ERR_NOT_IMPLEMENTED = 6
} o3g_status;

enum { O3G_FLAG_NO_CORRESPONDENCES = 1, O3G_FLAG_DEGENERATE = 2,
       O3G_FLAG_COMM_TIMEOUT = 4 /* peer-memory exchange: a rank's partial never arrived; the loop
                                    stopped with the last T (o3g_dist_peer_connect) */ };

/* Number of reduction terms of one pass (R4):
 * [0..20] J^T J upper triangle, row-major (i <= j); [21..26] J^T r;
 * [27] inlier count; [28] sum of squared Euclidean distances d^2.       */
#define O3G_NTERMS 29

typedef struct {
    int32_t iterations;  /* Gauss-Newton updates applied (<= max_iterations) */
    int32_t passes;      /* correspondence passes run = iterations + 1 */
    int32_t converged;   /* 1 if the S:285 criteria stopped the loop */
    int32_t flags;       /* O3G_FLAG_* */
    double fitness;      /* at T_out: inliers / n_source */
    double inlier_rmse;  /* at T_out: sqrt(sum d^2 / inliers), 0 if none */
    double inlier_count; /* at T_out */
} o3g_icp_info;

typedef struct o3g_ctx o3g_ctx;

/* ---------------------------------------------------------------- one-shot
 * registration_icp, point-to-plane.
 * source_xyz [n_source][3], target_xyz / target_normals [n_target][3]:
 * float32, host or device. Normals are used as given (R10).
 * max_correspondence_distance: the inclusive radius dmax (R1).
 * max_iterations: number of updates (>= 0). relative_fitness,
 * relative_rmse: absolute-difference thresholds between consecutive passes
 * with strict '<' (R8). Outputs (host): T_out[16], *fitness, *inlier_rmse,
 * info (nullable). Uses a per-thread cached context on the current device.
 */
o3g_status o3g_icp_point_to_plane(const float* source_xyz, int64_t n_source,
                                  const float* target_xyz, const float* target_normals,
                                  int64_t n_target, const double init_T[16],
                                  double max_correspondence_distance, int32_t max_iterations,
                                  double relative_fitness, double relative_rmse, double T_out[16],
                                  double* fitness, double* inlier_rmse, o3g_icp_info* info,
                                  void* cuda_stream);

/* registration_icp with TransformationEstimationPointToPoint(False)
 * (SPEC S:255-263): same arguments, loop,
 * criteria, flags and return values as o3g_icp_point_to_plane, no normals. */
o3g_status o3g_icp_point_to_point(const float* source_xyz, int64_t n_source,
                                  const float* target_xyz, int64_t n_target,
                                  const double init_T[16], double max_correspondence_distance,
                                  int32_t max_iterations, double relative_fitness,
                                  double relative_rmse, double T_out[16], double* fitness,
                                  double* inlier_rmse, o3g_icp_info* info, void* cuda_stream);

/* --------------------------------------------------------------- stateful */
/* Create a context on CUDA device `device`, ordered on `cuda_stream`.     */
o3g_status o3g_create(o3g_ctx** out, int device, void* cuda_stream);
o3g_status o3g_destroy(o3g_ctx* ctx);

/* A1: build the voxel-hash grid over the target (cell size
 * dmax*(1+2^-20)); keeps sorted float4 copies of xyz (+ original index)
 * and normals. normals may be NULL only for point-to-point estimation.
 * Invalidates any previously set source ordering.                       */
o3g_status o3g_set_target(o3g_ctx* ctx, const float* xyz, const float* normals, int64_t n,
                          double max_correspondence_distance);

/* A2: store the source, ordered by the grid cell of order_T * s (NULL =
 * identity) for locality. Requires o3g_set_target first. The FULL source
 * is passed on every rank; when distributed (o3g_dist_init) the context
 * keeps its contiguous shard of the spatial order and the fitness
 * denominator stays n (the global count). 1 <= n <= 2^31 - 2^24 (the
 * kernels' 32-bit batch cursors step past the last query); device arrays
 * must live on the context's device (O3G_ERR_INVALID_ARGUMENT otherwise). */
o3g_status o3g_set_source(o3g_ctx* ctx, const float* xyz, int64_t n, const double order_T[16]);

/* A1 + A2 in one call: o3g_set_target(target_xyz, target_normals, n_target,
 * dmax) followed by o3g_set_source(source_xyz, n_source, order_T), same
 * arguments, results and errors (this is what o3g_icp_point_to_plane does
 * with its clouds). With device-resident arrays on a single GPU the source's
 * bbox, ordering keys, sort and gather only need the grid's dimensions, so
 * they run on a second stream with their own scratch beside the target's
 * sort, cell table, gather and bitmaps, and the call waits once for both;
 * host arrays are staged with their copies overlapped with the build.      */
o3g_status o3g_set_clouds(o3g_ctx* ctx, const float* source_xyz, int64_t n_source,
                          const float* target_xyz, const float* target_normals, int64_t n_target,
                          double max_correspondence_distance, const double order_T[16]);

/* One correspondence + reduction pass at fixed T_in (north_star's
 * o3g_icp_step). Outputs:
 *   corr_out: DEVICE int32 [n] or NULL. Written in ORIGINAL source order
 *     with ORIGINAL target indices; -1 = no target within dmax. When
 *     distributed, only this rank's shard positions are written.
 *   JTJ_out[36] (full symmetric, mirrored from 21 terms), JTr_out[6],
 *   *inlier_count, *sum_sq_dist: host, nullable; summed over all ranks.
 *   terms_out[O3G_NTERMS]: host, nullable, the raw 29 terms.             */
o3g_status o3g_icp_step(o3g_ctx* ctx, const double T_in[16], int32_t* corr_out,
                        double JTJ_out[36], double JTr_out[6], double* inlier_count,
                        double* sum_sq_dist, double* terms_out);

/* The full loop on device (CUDA graph of max_iterations+1 passes, T and the
 * criteria state resident in device memory; one host sync at the end).
 * hist_fitness / hist_rmse: host, nullable, capacity max_iterations+1,
 * one entry per pass.                                                   */
o3g_status o3g_icp_run(o3g_ctx* ctx, const double init_T[16], int32_t max_iterations,
                       double relative_fitness, double relative_rmse, double T_out[16],
                       double* fitness, double* inlier_rmse, o3g_icp_info* info,
                       double* hist_fitness, double* hist_rmse);

/* --------------------------------------------------- normal estimation
 * estimate_normals ("KDTreeSearchParamHybrid(
 * radius = 0.1, max_nn = 30)"): for every point, the hybrid
 * neighbourhood is the min(max_nn, count) nearest points within radius
 * (the point itself included; the ICP pass's exact fp64 distance rule,
 * inclusive, ties -> lower index); mean and covariance in fp64 in (d^2,
 * index) order; normal = unit eigenvector of the smallest eigenvalue with
 * its largest-magnitude component positive; < 3 neighbours -> (0,0,1),
 * counted in *n_fallback. xyz: [n][3] float32 host or device, n >= 3;
 * 1 <= max_nn <= 64. out_normals: DEVICE float32 [n][3]; nbr_count:
 * DEVICE int32 [n] or NULL. Builds the cloud's grid in the context (it
 * REPLACES the context's target; call o3g_set_target again afterwards).  */
o3g_status o3g_estimate_normals(o3g_ctx* ctx, const float* xyz, int64_t n, double radius,
                                int32_t max_nn, float* out_normals, int32_t* nbr_count,
                                int64_t* n_fallback);

/* ------------------------------------------------ batched evaluation
 * evaluate_registration (the RANSAC validation step the
 * paper profiles as its most time-consuming part) for k
 * transforms at once: for each Ts[16 i .. 16 i + 15] (host, row-major,
 * rigid) fitness[i] = inliers / n and inlier_rmse[i] = sqrt(sum d^2 /
 * inliers) (0 if none) with exactly the correspondence rule of the ICP
 * pass, no re-estimation. Uses the context's target and source; one
 * launch covers all k (grid.y = transform). 1 <= k <= 65535. Single GPU
 * (O3G_ERR_NOT_IMPLEMENTED when distributed).                           */
o3g_status o3g_evaluate_registration(o3g_ctx* ctx, const double* Ts, int32_t k, double* fitness,
                                     double* inlier_rmse);

/* ------------------------------------------- downsampling and multi-scale
 * voxel_down_sample (Fig. 1): each output point
 * is the mean of the input points of one occupied voxel of the grid anchored
 * at the cloud's minimum bound, index floor((p - min) / voxel) per axis;
 * normals (nullable) are averaged the same way and renormalised (a zero sum
 * stays zero); output in ascending lexicographic (ix, iy, iz) order.
 * Sums are fp64 in original-index order, the mean is rounded once to fp32.
 * xyz / normals: [n][3] float32, host or device. out_xyz / out_normals:
 * DEVICE float32 [n][3] capacity (out_normals may be NULL). *n_out: host.
 * O3G_ERR_INVALID_ARGUMENT for n <= 0, voxel <= 0 or non-finite input, or
 * more than 2^63 voxels in the bounding box.                            */
o3g_status o3g_voxel_down_sample(o3g_ctx* ctx, const float* xyz, const float* normals, int64_t n,
                                 double voxel, float* out_xyz, float* out_normals, int64_t* n_out);

/* Multi-scale point-to-plane ICP (BASELINE config 4):
 * for s = 0..n_scales-1, downsample source and target (with normals) at
 * voxel[s], run the loop of o3g_icp_run with max_correspondence_distance
 * dmax[s] and max_iterations iters[s] starting from the current T, and
 * carry T to the next scale (R13). Arrays of length n_scales are
 * host memory; the per-scale outputs (nullable) receive fitness, inlier
 * rmse, updates applied and the downsampled source size of each scale.   */
o3g_status o3g_icp_multiscale(o3g_ctx* ctx, const float* source_xyz, int64_t n_source,
                              const float* target_xyz, const float* target_normals,
                              int64_t n_target, const double init_T[16], int32_t n_scales,
                              const double* voxel, const double* dmax, const int32_t* iters,
                              double relative_fitness, double relative_rmse, double T_out[16],
                              double* fitness_per_scale, double* rmse_per_scale,
                              int32_t* iterations_per_scale, int64_t* n_source_per_scale);

/* ------------------------------------------------------------ multi-GPU
 * One process per GPU. Rank 0 calls o3g_nccl_unique_id (128 bytes), the
 * caller broadcasts it (e.g. torch.distributed), every rank calls
 * o3g_dist_init before o3g_set_source. Each pass then all-gathers the 29
 * partial terms of every rank (232 B + padding per rank) and sums them in
 * rank order on every rank, so T is bit-identical everywhere.
 * NCCL is loaded at run time (libnccl.so.2); O3G_ERR_COMM if unavailable.
 * world == 1 with a NULL id is the single-GPU path; world == 1 WITH an id
 * creates a one-rank communicator and runs the distributed pass (rank slot,
 * graph-captured ncclAllGather, rank-order tail) on one GPU — a self-test of
 * the NCCL leg; results equal the single-GPU path's.                      */
o3g_status o3g_nccl_unique_id(void* id_out_128);
o3g_status o3g_dist_init(o3g_ctx* ctx, int rank, int world, const void* nccl_unique_id_128);

/* Peer-memory exchange (SURVEY §8(e) "fused one-shot exchange"; replaces the
 * per-pass NCCL all-gather): each rank owns a small exchange buffer in device
 * memory; the last block of a rank's correspondence kernel stores its 29-term
 * partial straight into EVERY rank's buffer (peer stores over NVLink) and
 * releases a per-pass epoch flag there; the rank's tail kernel acquires the
 * world flags of its own buffer, sums the slots in rank order and runs the A8
 * update — two kernels per pass, no collective call, T bit-identical on every
 * rank as with the all-gather. Setup (after o3g_dist_init with world > 1, all
 * ranks on one node with peer access): every rank calls o3g_dist_peer_handle
 * (64 bytes out, host: the CUDA IPC handle of its buffer), the caller
 * all-gathers the handles (e.g. torch.distributed) and every rank passes the
 * world x 64 bytes (rank order) to o3g_dist_peer_connect. Every rank must make
 * the same sequence of step/run calls (the epochs count them). A rank whose
 * peers never arrive stops after 20 s with O3G_FLAG_COMM_TIMEOUT instead of
 * hanging. O3G_ERR_COMM if a handle cannot be opened (no peer access);
 * o3g_dist_init drops the connection.                                     */
#define O3G_PEER_HANDLE_BYTES 64
o3g_status o3g_dist_peer_handle(o3g_ctx* ctx, void* handle_out_64);
o3g_status o3g_dist_peer_connect(o3g_ctx* ctx, const void* handles_world_x_64);

/* In-process loopback of the multi-GPU path (verification of SURVEY §8(e)
 * A7 on one device): o3g_dist_init_loopback makes ctx rank `rank` of `world`
 * WITHOUT a communicator (call it before o3g_set_source, which then keeps the
 * rank's contiguous shard); o3g_loopback_run drives the world contexts
 * ctxs[0..world) (ctxs[r] of rank r, all on the same device, same target,
 * source and options) pass by pass in lockstep on ctxs[0]'s stream: every
 * rank's correspondence kernels on its shard, its TAIL_WRITE_RANK tail, the
 * exchange of the world x 29 partial terms (device copies in place of the
 * NCCL all-gather), and every rank's TAIL_SUM_RANKS tail (rank-order sum +
 * the A8 update) — the kernels of the distributed path, only the transport
 * differs. Outputs as o3g_icp_run, from rank 0; O3G_ERR_CUDA if the ranks'
 * transforms ever differ (they must be bit-identical). o3g_last_run_trace
 * works on each context afterwards.                                      */
o3g_status o3g_dist_init_loopback(o3g_ctx* ctx, int rank, int world);
/* Loopback with the peer-memory exchange: wires the world loopback contexts'
 * exchange buffers to one another (plain device pointers instead of IPC
 * mappings); o3g_loopback_run then runs every rank's publishing kernels
 * before any rank's waiting tail, so the waits are already satisfied and no
 * kernel on the device ever waits for a later one.                        */
o3g_status o3g_loopback_peer_connect(o3g_ctx* const* ctxs, int world);
o3g_status o3g_loopback_run(o3g_ctx* const* ctxs, int world, const double init_T[16],
                            int32_t max_iterations, double relative_fitness, double relative_rmse,
                            double T_out[16], double* fitness, double* inlier_rmse, o3g_icp_info* info);

/* -------------------------------------------------------------- options
 * O3G_OPT_SEARCH: correspondence-kernel variant, all bit-identical
 *   (DESIGN.md §5): 0 = exact fp64 test of every candidate; 1 = two-pass
 *   warp kernel (fp32 prefilter with a proven margin + exact fp64 decision;
 *   the default); 2 = single-pass fp32 prefilter + exact decision; 3 =
 *   two-pass kernel on count-sorted 128-query tiles; 4 = two-pass kernel on
 *   tiles of <= 128 queries (source in 8^3-brick Morton order, set at the next
 *   o3g_set_source) whose target neighbourhood is staged in shared memory
 *   (dense grid; a hashed grid runs variant 1). Point-to-point estimation and
 *   batched evaluation always run variant 1.
 * O3G_OPT_GRID: 0 = auto, 1 = force dense cell table, 2 = force hashed
 *   cell table (collisions only add candidates; results are identical).
 * O3G_OPT_TIMING: 1 = record CUDA events around every correspondence
 *   kernel inside the run graph (read with o3g_last_run_kernel_ms).
 * O3G_OPT_BLOCKS_PER_SM: override the persistent grid size (0 = auto).
 * O3G_OPT_NBR_MASK: 1 = skip queries whose 27-cell stencil is empty using a
 *   dilated occupancy bitmap of the dense grid (default), 0 = off.
 * O3G_OPT_COOP_MIN: variant 1 scans a query with at least this many
 *   candidates with the whole warp (0 = never; -1 = auto, the default:
 *   32 when the target averages >= 32 points per occupied cell, else 0).
 * O3G_OPT_ESTIMATION: 0 = point-to-plane (default), 1 = point-to-point
 *   (TransformationEstimationPointToPoint(False); SPEC
 *   S:255-263): Horn's closed-form rigid fit on the correspondences, no
 *   scale, det R = +1; degenerate if < 3 pairs or rank(H) < 2 (R15). The
 *   29 terms of o3g_icp_step then hold [0..8] sum s'q^T (row-major),
 *   [9..11] sum s', [12..14] sum q, [27] count, [28] sum d^2 (JTJ/JTr
 *   outputs carry the same raw slots). Target normals are then optional.
 * O3G_OPT_SOURCE_ORDER: order of the source copy (locality only): 0 = by
 *   the target grid's cell index of order_T s (default), 1 = Morton order of
 *   4x4x4-cell bricks (takes effect at the next o3g_set_source).
 * O3G_OPT_TARGET_SORT: how o3g_set_target orders the target by cell: 0 =
 *   counting sort (histogram, scan, atomic scatter), 1 = stable radix sort
 *   of (cell, index) + gather (default; 1.8 ms faster per 16M-point build).
 *   Only the order inside a cell differs; every consumer breaks ties by the
 *   original index.
 * O3G_OPT_PRUNE_MIN: variant 1, dense grid: a query with at least this
 *   many candidates first scans one x-row, then skips the rows whose lower
 *   distance bound exceeds that row's best; -1 = auto
 *   (default: for targets averaging >= 4 points per occupied cell, the
 *   pruning kernel without the light-query pre-scan — the run loop's warm
 *   start prunes every pass after the first and cuts end cells of rows —
 *   and, at >= 32, the cooperative path's row pruning; else off),
 *   -2 = never, 0 = every query. Independently, o3g_icp_run's passes after
 *   the first bound every query by its previous winner (warm start).
 *   Results are identical either way.
 * O3G_OPT_INTERLEAVE: variant 1 batch composition: 0 = 32 consecutive
 *   queries of the ordered source per warp batch; 1 = lane l of batch b
 *   takes query l * ceil(n/32) + b (spreads clustered heavy queries over
 *   all warps); -1 = auto (default: on when the cooperative path is).
 * O3G_OPT_XSORT: order the target by x inside each cell (set at the next
 *   o3g_set_target) so the cooperative path scans, per x-row, only the
 *   window |q_x - s'_x| <= sqrt(ub - L) found by a warp-wide search
 *   (DESIGN.md §5.2c); -1 = auto (default: >= 32 points per occupied cell).
 * O3G_OPT_CERT: correspondence certificates in o3g_icp_run (variant 1;
 *   DESIGN.md §5.5): each full search leaves a per-query radius rho such
 *   that its answer provably holds while the transformed query moves by
 *   less than rho (half the gap between the nearest and second-nearest
 *   target, or the clearance beyond dmax when there is no winner); later
 *   passes check the displacement |(T_k - T_b) s| against rho and search
 *   only the queries whose certificate expired. A pass runs this way once the
 *   previous pass matched more than half of the source (the refinement
 *   phase); earlier passes run the plain search. -1 = auto (default: shards
 *   of >= 2^20 queries), 1 = on, 0 = off (the previous winner then only
 *   bounds the next search, the warm start), 2 = on from the second pass
 *   regardless of fitness (experiments).
 * O3G_OPT_CERT_SWEEP: how a certificate pass settles the certified queries:
 *   0 = inside the search kernel's pre-pass (fused; default), 1 = a separate
 *   streaming sweep kernel that flags the rest for the search (experiments).
 * O3G_OPT_TRACE_PASS: k >= 0 = o3g_icp_run also writes the correspondences
 *   of pass k (original source order) for o3g_last_run_trace; -1 = off
 *   (default). A testing hook: it adds a scattered index write to pass k.
 * Results are identical for every value of the other options.           */
enum { O3G_OPT_SEARCH = 1, O3G_OPT_GRID = 2, O3G_OPT_TIMING = 3, O3G_OPT_BLOCKS_PER_SM = 4,
       O3G_OPT_NBR_MASK = 5, O3G_OPT_COOP_MIN = 6, O3G_OPT_ESTIMATION = 7,
       O3G_OPT_SOURCE_ORDER = 8, O3G_OPT_TARGET_SORT = 9, O3G_OPT_PRUNE_MIN = 10,
       O3G_OPT_INTERLEAVE = 11, O3G_OPT_XSORT = 12, O3G_OPT_CERT = 13, O3G_OPT_TRACE_PASS = 14,
       O3G_OPT_CERT_SWEEP = 15 };
o3g_status o3g_set_option(o3g_ctx* ctx, int option, int64_t value);

/* Sum of the correspondence-kernel (K3) durations of the last o3g_icp_run
 * with O3G_OPT_TIMING=1, the number of K3 launches that did work, and the
 * tail-kernel total. Milliseconds.                                      */
o3g_status o3g_last_run_kernel_ms(o3g_ctx* ctx, double* k3_ms, int32_t* k3_launches,
                                  double* tail_ms);

/* Per-pass record of the last o3g_icp_run (verification hook, the run-loop
 * analogue of o3g_icp_step): T_hist [passes][16] the T each pass ran with,
 * terms_hist [passes][O3G_NTERMS] that pass's 29 terms (same layout as
 * o3g_icp_step's terms_out), and corr_out [n_source] the correspondences of
 * pass O3G_OPT_TRACE_PASS in original source order (-1 = none; host or
 * device memory; untouched if that pass did not run), and stats_hist
 * [passes][3] per pass: the queries that ran the full correspondence search,
 * the candidates those searches scanned, and the queries settled by a valid
 * certificate (the rest had an empty 27-cell stencil) (variant 1; 0 for the
 * other variants).
 * passes = info.passes of that run; on a multi-GPU context corr_out holds
 * this rank's shard only (other entries -2) and stats_hist this rank's
 * counts. Any pointer may be NULL.                                         */
o3g_status o3g_last_run_trace(o3g_ctx* ctx, double* T_hist, double* terms_hist, int32_t* corr_out,
                              double* stats_hist);

/* Grid statistics of the current target: cells per axis, table entries,
 * hashed (0/1), occupied cells. Any pointer may be NULL.                 */
o3g_status o3g_grid_info(o3g_ctx* ctx, int64_t dims[3], int64_t* table_size, int32_t* hashed,
                         int64_t* occupied_cells);

/* Kernel launches issued by this context so far (all kinds).            */
int64_t o3g_launch_count(const o3g_ctx* ctx);

const char* o3g_status_string(o3g_status s);
/* Last error message of the calling thread ("" if none).                */
const char* o3g_last_error(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* O3G_H */
