// o3g_internal.cuh — shared declarations of the CUDA library (not installed).
// Device data layout and kernel entry points; see DESIGN.md §4-§5.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace o3g {

constexpr int kTerms = 29;        // O3G_NTERMS
constexpr int kTermStride = 32;   // padded per-block / per-rank partial
// per-pass statistics ride in the padding (variant 1; others leave them 0):
// [29] queries that ran the full search, [30] candidates they scanned, [31]
// queries settled by a valid certificate (k3_sweep)
constexpr int kStatSearched = 29, kStatCandidates = 30, kStatCertified = 31, kTermsStats = 32;
#ifndef O3G_K3_THREADS
#define O3G_K3_THREADS 256
#endif
constexpr int kK3Threads = O3G_K3_THREADS;   // correspondence kernel block size
constexpr int kTailThreads = 1024;

// Voxel-hash grid over the target. Cell size
// h = dmax*(1+2^-20) so the 27-cell stencil provably contains every target
// within dmax of a query. table index of cell (cx,cy,cz):
//   dense : (cz*ny + cy)*nx + cx            (collision-free)
//   hashed: (rowhash(cy,cz) + cx) & hmask   (collisions only add candidates)
// Along x consecutive cells map to consecutive table entries in both modes,
// so the 3 cells of one x-row are one contiguous range of the sorted target
// (two if a hashed row wraps).
struct GridDev {
    double ox, oy, oz;   // componentwise min of the target (fp32 values)
    double inv_h;        // 1 / h
    int32_t nx, ny, nz;  // cells per axis
    int32_t hashed;
    uint32_t hmask;      // table_size - 1 when hashed
    int32_t pad;
    int64_t table_size;  // cell_start has table_size + 1 entries
    double h;            // cell edge dmax (1 + 2^-20) (row lower bounds, k3_balanced)
};

// Loop state, resident in device memory for the whole graph-launched loop.
struct IcpState {
    double T[16];
    double terms[kTermStride];
    double fit, rmse, fit_prev, rmse_prev;
    double rel_fit, rel_rmse;
    double n_total;
    int32_t it, max_it, passes, done, flags, converged, hist_cap;
    int32_t cmode;   // certificates: this pass runs the sweep + certified search (set by
                     // the previous pass's tail: fitness > 1/2, the refinement phase)
    int32_t cforce;  // O3G_OPT_CERT = 2: every pass after the first (experiments)
    int32_t gbase;   // certificates carry (gbase + pass) mod 2^16: a record from an earlier
                     // run is older than the current pass index, hence invalid; the host
                     // advances gbase per run and requests a reset (creset) on wrap-around
    int32_t creset;  // 1: k_cert_reset clears the records at the head of this run
    uint32_t xbase;  // peer-memory exchange: pass p of this run carries epoch xbase + p + 1
                     // (the host advances it per run, identically on every rank)
};

// Peer-memory exchange buffer of one rank (TAIL_PEER; SURVEY §8(e) "fused
// one-shot exchange"): rank r's last K3 block stores its 32-slot partial into
// slots[epoch & 1][r] of EVERY rank's buffer (peer stores over NVLink), then
// releases flags[epoch & 1][r] = epoch there; the rank's tail kernel acquires
// its own world flags and sums the slots in rank order. Two parities: a rank
// can run at most one pass ahead of the slowest reader (its pass p + 2 needs
// every rank's flag of pass p + 1, set after that rank's tail of pass p).
constexpr int kMaxWorld = 64;
struct Xchg {
    double slots[2][kMaxWorld][kTermStride];
    unsigned int flags[2][kMaxWorld];
};

enum TailMode : int {
    TAIL_REDUCE_BLOCKS = 1,  // terms = fixed-order sum of the K3 block partials
    TAIL_WRITE_RANK = 2,     // store terms into gathered[rank] and stop
    TAIL_SUM_RANKS = 4,      // terms = sum over gathered[0..world) in rank order
    TAIL_SOLVE = 8,          // criteria + LDLT + exp + T update (A8)
    TAIL_STEP = 16,          // store terms only (o3g_icp_step)
    TAIL_P2P = 32,           // point-to-point estimation (Horn's quaternion fit)
    TAIL_PEER = 64,          // rank exchange through peer memory (Xchg) instead of gathered[]:
                             // WRITE_RANK publishes to every rank, SUM_RANKS waits for all flags
};

__host__ __device__ inline int64_t grid_index_dense(const GridDev& g, int cx, int cy, int cz) {
    return ((int64_t)cz * g.ny + cy) * (int64_t)g.nx + cx;
}
__host__ __device__ inline uint32_t grid_row_hash(int cy, int cz) {
    return (uint32_t)cy * 0x9E3779B1u ^ (uint32_t)cz * 0x85EBCA77u ^ 0x27D4EB2Fu;
}

#ifdef __CUDACC__
// Cell coordinate floor((x - o) / h), computed as floor((x - o) * inv_h) in
// fp64 without contraction; clamped to [-2, n+1] so far queries cannot
// overflow (they have no candidates anyway). Used identically for the
// target points (grid build) and the transformed queries (search).
// (cvt.rmi.s32.f64 floors and saturates out-of-range values, then the int
// clamp; identical to clamping in fp64 first for every finite x.)
__device__ __forceinline__ int cell_coord(double x, double o, double inv_h, int n) {
    const int c = __double2int_rd(__dmul_rn(__dsub_rn(x, o), inv_h));
    return min(max(c, -2), n + 1);
}

// A3: s' = T s, fixed order ((T00 sx + T01 sy) + T02 sz) + T03, no FMA (R2).
__device__ __forceinline__ void xform_rn(const double* T, float x, float y, float z, double& ox,
                                         double& oy, double& oz) {
    const double dx = x, dy = y, dz = z;
    ox = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[0], dx), __dmul_rn(T[1], dy)), __dmul_rn(T[2], dz)), T[3]);
    oy = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[4], dx), __dmul_rn(T[5], dy)), __dmul_rn(T[6], dz)), T[7]);
    oz = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(T[8], dx), __dmul_rn(T[9], dy)), __dmul_rn(T[10], dz)), T[11]);
}
#endif

// ---- launchers (grid_build.cu)
void launch_bbox(const float* xyz, int64_t n, uint32_t* minmax6, int32_t* nonfinite, int sms,
                 cudaStream_t s);
void launch_check_finite(const float* v, int64_t count, int32_t* nonfinite, int sms,
                         cudaStream_t s);
// brick = 1: Morton order of 4x4x4-cell bricks (source ordering only;
// needs < 2^10 bricks per axis), 0: the table index
void launch_cell_keys(const float* xyz, int64_t n, const GridDev& g, const double* T12_or_null,
                      uint32_t* keys, int32_t* vals, cudaStream_t s, int brick = 0);
void launch_cs_runs(const uint32_t* keys, int64_t n, int32_t* runs, uint32_t* occ_bits, cudaStream_t s);
// cell start table [cells + 1] from the sorted keys in one pass (+ occupancy bits)
void launch_cs_fill(const uint32_t* keys, int64_t n, int64_t cells, int32_t* cs, uint32_t* occ_bits,
                    cudaStream_t s);
void launch_dilate3(uint32_t* bits, uint32_t* tmp, int64_t ncells, int64_t nx, int64_t nxny, cudaStream_t s);
void launch_coarse_bits(const float4* tpos, int64_t n, const GridDev& g, int shift, int cnx, int cny,
                        uint32_t* bits, cudaStream_t s);
void launch_xkeys(const float4* tpos, int64_t n, const GridDev& g, uint64_t* keys, int32_t* vals,
                  cudaStream_t s);
void launch_permute_target(const float4* tpos, const float4* tnrm, const int32_t* perm, int64_t n,
                           float4* opos, float4* onrm, cudaStream_t s);
void launch_run_marks(const uint32_t* keys, int64_t n, int shift, int32_t* mark, cudaStream_t s);
void launch_tile_flags(const int32_t* run_start, int64_t n, int tq, uint8_t* flag, cudaStream_t s);
void launch_histogram(const uint32_t* keys, int64_t n, int32_t* counts, unsigned long long* occupied,
                      cudaStream_t s);
void launch_scatter_target(const float* xyz, const float* nrm, const uint32_t* keys, int64_t n,
                           int32_t* cursor, float4* tpos, float4* tnrm, cudaStream_t s);
void launch_gather_target(const float* xyz, const float* nrm, const int32_t* vals_sorted,
                          const uint32_t* keys_sorted, int64_t n, float4* tpos, float4* tnrm,
                          unsigned long long* occupied, cudaStream_t s);
constexpr int kShardBuckets = 4096;   // (grid_build.cu) source-shard histogram buckets
void launch_key_hist(const uint32_t* keys, int64_t n, int shift, int nx, const uint32_t* live, uint32_t* hist,
                     int sms, cudaStream_t s);
void launch_key_flags(const uint32_t* keys, int64_t n, int shift, int nx, uint32_t blo, uint32_t bhi,
                      uint8_t* flags, cudaStream_t s);
void launch_gather_source(const float* xyz, const int32_t* vals_sorted, int64_t lo, int64_t hi,
                          float4* out, cudaStream_t s);
void launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t s);
void launch_cert_reset(float4* cert, int64_t n, const IcpState* st, cudaStream_t s);
// dilated occupancy bitmap of a dense grid: occupancy from cell_start, then
// three shifted-OR passes (x by 1, y by nx, z by nx*ny). Bits that wrap across
// row / slab boundaries only add false positives (a query then just does the
// full search). Result in `out` (words = ceil(ncells / 32)).
void launch_nbr_bits(const int32_t* cell_start, int64_t ncells, int64_t nx, int64_t nxny,
                     uint32_t* tmp, uint32_t* out, cudaStream_t s);

// ---- launchers (voxel.cu)
void launch_vox_keys(const float* xyz, int64_t n, const double mn[3], double voxel, uint64_t dy,
                     uint64_t dz, uint64_t* keys, int32_t* vals, cudaStream_t s);
void launch_run_flags(const uint64_t* keys, int64_t n, int32_t* flags, cudaStream_t s);
void launch_run_starts(const int32_t* flags, const int32_t* runid, int64_t n, int32_t* starts,
                       cudaStream_t s);
void launch_vox_mean(const float* xyz, const float* nrm, const int32_t* vals, const int32_t* starts,
                     int64_t nruns, float* out_xyz, float* out_nrm, cudaStream_t s);

// ---- launchers (normals.cu)
void launch_normals(const float4* tpos, int n, const int32_t* cs, const GridDev& g, double r2,
                    int max_nn, float* out, int32_t* nbr_count, unsigned long long* fallback,
                    cudaStream_t s);

// ---- launchers (icp_kernels.cu)
struct K3Args {
    const float4* src;      // sorted local shard (x,y,z, bitcast original index)
    int32_t n;              // local count
    const float4* tpos;     // sorted target (x,y,z, bitcast original index)
    const float4* tnrm;     // sorted target normals (nx,ny,nz,0)
    const int32_t* cell_start;
    GridDev g;
    double r2;              // dmax*dmax (fp64, R1)
    double dmax, inv_dmax;  // prefilter margin terms
    const IcpState* st;
    double* block_partials; // [gridDim.x][kTermStride]
    int32_t* corr_out;      // original order, nullable
    const uint32_t* nbr_bits;  // dense grid: bit k set iff some cell of k's 27-stencil
                               // is occupied (a conservative skip test); hashed grid:
                               // the same over 2^cshift-cell coarse cells; nullable
    int cshift, cnx, cny;      // hashed grid: coarse cell = cell >> cshift, dims
    int p2p;                   // record = point-to-point terms (sum s'q^T, sum s', sum q)
    int n_eval;
    const double* eval_T;      // batched evaluation: T of blockIdx.y is eval_T[16 * y]
                               // (nullable); partials at [(y * gridDim.x + x) * 32]
    int coop_min;              // variant 1: queries with >= coop_min candidates are
                               // scanned by the whole warp (0 = never)
    const int32_t* tiles;      // variant 4: tile starts in the local source (ntiles)
    int32_t ntiles;
    int ilv;                   // variant 1: 0, or interleaved batches (= ceil(n / 32))
    int32_t* prev_j;           // variant 1 run loop without certificates: per local query,
                               // the previous pass's winner (sorted target position, -1
                               // none); nullable
    // correspondence certificates (variant 1 run loop): per local
    // query i a 32-byte record cert[2i] = {bits(winner j (sorted position) or -1),
    // bits((cert pass << 16) | half(rho / h)), q.x, q.y}, cert[2i+1] = {q.z, n.x,
    // n.y, n.z} (the winner's position and normal, cached: a certified query
    // streams 32 B and gathers nothing). The result of pass b stays exact at a
    // later pass while the query has moved by less than rho since pass b.
    // nullable (= off). With certificates a pass is two kernels: k3_sweep
    // settles every certified (or bitmap-dead) query and flags the rest in
    // need[i]; k3_balanced then searches only the flagged ones.
    float4* cert;
    uint8_t* need;             // k3_sweep -> k3_balanced: 1 = run the full search
    int part_off;              // this kernel's first block-partial slot
    int part_total;            // fused tail: block partials to reduce (all kernels of the pass)
    double rhog_mul, rhog_cap; // certificate goal: min(mul x last pass's displacement bound, cap x h)
    int pass_expect;           // run loop: the pass this launch belongs to (-1: no check); a
                               // kernel finding IcpState::passes != pass_expect exits (the
                               // pass's other search instantiation already ran its tail)
    const uint32_t* nbr2_bits; // dense grid: the occupancy bitmap dilated twice (bit k set
                               // iff some cell within Chebyshev distance 2 is occupied)
    const double* hist_Tr;     // [pass][16]: the T each pass ran with (certificate ages)
    float smax[3];             // max |source coordinate| per axis (displacement bound)
    float h_rd, inv_h_rd;      // cell edge h and 1/h, rounded down (rho packing)
    int xsorted;               // target x-sorted inside cells: x-windows in the cooperative path
    int prune;                 // variant 1: row-pruning instantiation (dense grid)
    int prune_min;             //   ... for light queries with >= prune_min candidates
    // fused tail (variant 1): the last block to finish reduces the block
    // partials in fixed order and runs the A8 epilogue (mode = TAIL_*), or,
    // distributed, writes the rank's slot for the exchange
    int fuse_mode;             // 0 = separate k_tail launch
    unsigned int* counter;     // zero between launches (the last block resets it)
    IcpState* st_rw;
    double* hist_fit;
    double* hist_rmse;
    double* hist_T;            // per pass: T used and the 29 terms (nullable)
    double* hist_terms;
    // (world > 1, fuse_mode & TAIL_WRITE_RANK) the last block stores the
    // rank's 32-slot partial at gathered[rank] instead of finishing the pass
    double* gathered;
    int rank;
    // (fuse_mode & TAIL_PEER) peer-memory exchange: xpeers[q] = rank q's Xchg
    // (this rank's own buffer at [rank]; a device array of world pointers)
    Xchg* const* xpeers;
    int world;
    int nt;   // variant 1: threads per block (256, 512 or 1024; k3_balanced_threads)
};
constexpr int kCertAges = 32;     // certificates older than this many passes expire
// variant: 0 = exact fp64 scan (k3_corr_reduce), 1 = two-pass warp kernel
// (k3_balanced, the default), 2 = single-pass prefilter (k3_corr_reduce<true>),
// 3 = tile-sorted two-pass kernel (k3_sorted), 4 = smem-staged tiles (k3_tiled).
// Identical correspondences.
constexpr int kTileQ = 128;       // variant 4: queries per tile (max)
// variant 1's block size (K3Args::nt): 1024 threads (one block per SM) for shards of
// >= 2^19 queries, 512 below (measured: large16m K3 0.601 ms at 256, 0.593 at 512,
// 0.559 at 1024; depth 0.038 / 0.036 / 0.044; profiles/r02_cert_modes.txt)
inline int k3_balanced_threads(int64_t n_local) { return n_local >= (1 << 19) ? 1024 : 512; }
inline int k3_threads(int variant, int nt) { return variant == 3 ? 128 : variant == 4 ? kTileQ : variant == 1 ? nt : kK3Threads; }
int k3_tiled_blocks_per_sm(bool write_corr);
void launch_k3_tiled(const K3Args& a, int blocks, bool write_corr, cudaStream_t s);
int k3_sorted_blocks_per_sm(bool write_corr, int hashed);
void launch_k3_sorted(const K3Args& a, int blocks, bool write_corr, cudaStream_t s);
void launch_k3(const K3Args& a, int blocks, int variant, bool write_corr, cudaStream_t s);
int k3_sweep_blocks_per_sm();
void launch_k3_sweep(const K3Args& a, int blocks, bool write_corr, cudaStream_t s);
int k3_max_blocks_per_sm(int variant, bool write_corr, int hashed, bool prune, int nt);
void launch_eval_reduce(const double* partials, int nblocks, int k, double n_total, double* fit,
                        double* rmse, cudaStream_t s);
struct TailHist {
    double* fit;     // [pass]
    double* rmse;    // [pass]
    double* T;       // [pass][16], the T of the pass (before its update)
    double* terms;   // [pass][kTermStride]
};
void launch_tail(const double* block_partials, int nblocks, double* gathered, int world, int rank,
                 IcpState* st, TailHist hist, int mode, cudaStream_t s, Xchg* const* xpeers = nullptr);

}  // namespace o3g
