// grid_build.cu — per-call kernels of the hot path:
// target bounding box + finiteness check, cell keys, per-cell histogram
// (cell start table via exclusive scan), and the gathers that lay the sorted
// target / source out as float4 records for the correspondence kernel.
#include <float.h>

#include "o3g_internal.cuh"

namespace o3g {

// Order-preserving float <-> uint32 map, for atomicMin/atomicMax on floats.
__device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

// A0/A1: componentwise min/max of the target and a non-finite flag.
__global__ void k_bbox(const float* __restrict__ xyz, int64_t n, uint32_t* __restrict__ mm,
                       int32_t* __restrict__ nonfinite) {
    float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float v = xyz[3 * i + a];
            bad |= !finite_f(v);
            lo[a] = fminf(lo[a], v);
            hi[a] = fmaxf(hi[a], v);
        }
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        for (int o = 16; o; o >>= 1) {
            lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    // block reduce first: 6 atomics per block, not per warp (the per-warp
    // version serialised ~60k atomics on 6 words: 48 us for 2M points)
    __shared__ uint32_t s_mm[6];
    __shared__ int s_bad;
    if (threadIdx.x < 6) s_mm[threadIdx.x] = threadIdx.x < 3 ? 0xFFFFFFFFu : 0u;
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicMin(&s_mm[a], f2ord(lo[a]));
            atomicMax(&s_mm[3 + a], f2ord(hi[a]));
        }
        if (bad) s_bad = 1;
    }
    __syncthreads();
    if (threadIdx.x < 3) atomicMin(&mm[threadIdx.x], s_mm[threadIdx.x]);
    else if (threadIdx.x < 6) atomicMax(&mm[threadIdx.x], s_mm[threadIdx.x]);
    if (threadIdx.x == 0 && s_bad) atomicOr(nonfinite, 1);
}

__global__ void k_check_finite(const float* __restrict__ v, int64_t count, int32_t* nonfinite) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        bad |= !finite_f(v[i]);
    bad = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(nonfinite, 1);
}

// A1/A2: table index of the cell of each point (target: T = NULL, the raw
// coordinates; source: the cell of T s, clamped into the grid — ordering
// only, so clamping far points is harmless).
// spread the low 10 bits of v to every third bit (Morton interleave)
__device__ __forceinline__ uint32_t spread3(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_cell_keys(const float* __restrict__ xyz, int64_t n, GridDev g, bool has_T,
                            double T0, double T1, double T2, double T3, double T4, double T5,
                            double T6, double T7, double T8, double T9, double T10, double T11,
                            uint32_t* __restrict__ keys, int32_t* __restrict__ vals, int brick) {
    const double T[12] = {T0, T1, T2, T3, T4, T5, T6, T7, T8, T9, T10, T11};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
        double sx = x, sy = y, sz = z;
        if (has_T) xform_rn(T, x, y, z, sx, sy, sz);
        int cx = min(max(cell_coord(sx, g.ox, g.inv_h, g.nx), 0), g.nx - 1);
        int cy = min(max(cell_coord(sy, g.oy, g.inv_h, g.ny), 0), g.ny - 1);
        int cz = min(max(cell_coord(sz, g.oz, g.inv_h, g.nz), 0), g.nz - 1);
        uint32_t k;
        if (brick) {   // source order: Morton order of 2^b-cell bricks (b = brick), x-fastest inside
            const uint32_t b = (uint32_t)brick, m = (1u << b) - 1u;
            k = ((spread3((uint32_t)cx >> b) | (spread3((uint32_t)cy >> b) << 1) |
                  (spread3((uint32_t)cz >> b) << 2)) << (3 * b)) |
                (((uint32_t)cz & m) << (2 * b)) | (((uint32_t)cy & m) << b) | ((uint32_t)cx & m);
        } else {
            k = g.hashed ? ((grid_row_hash(cy, cz) + (uint32_t)cx) & g.hmask)
                         : (uint32_t)grid_index_dense(g, cx, cy, cz);
        }
        keys[i] = k;
        vals[i] = (int32_t)i;
    }
}

// cell starts from the radix-sorted keys: each occupied cell k records the end
// of its run (runs[k], zero elsewhere) and its occupancy bit; an exclusive max
// scan then gives cell c the end of the last occupied cell before c, i.e. the
// number of points with key < c (o3g_api.cu)
__global__ void k_cs_runs(const uint32_t* __restrict__ keys, int64_t n, int32_t* __restrict__ runs,
                          uint32_t* __restrict__ occ_bits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        if (i == n - 1 || keys[i + 1] != k) runs[k] = (int32_t)(i + 1);
        if (occ_bits && (i == 0 || keys[i - 1] != k)) atomicOr(&occ_bits[k >> 5], 1u << (k & 31));
    }
}

// The cell start table straight from the sorted keys, in one pass with no
// separate memset and max-scan: cs[c] = the first sorted position whose key is
// >= c, for c in [0, cells] (cs[cells] = n). Sorted position k (0..n) owns the
// cells (key[k-1], key[k]] (key[-1] = -1, key[n] = cells) and writes k into
// them; a warp takes 32 consecutive positions, each lane writes its own short
// range and the whole warp each long one (coalesced; long empty ranges do not
// serialise one thread). Also sets the occupancy bit of every occupied cell
// (dense grids).
__global__ void k_cs_fill(const uint32_t* __restrict__ keys, int64_t n, int64_t cells, int32_t* __restrict__ cs,
                          uint32_t* __restrict__ occ_bits) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 <= n; w += nwarps) {
        const int64_t k = w * 32 + lane;
        int64_t lo = 0, hi = -1;   // this lane's cells [lo, hi]
        if (k <= n) {
            const int64_t prev = k == 0 ? -1 : (int64_t)keys[k - 1];
            const int64_t cur = k == n ? cells : (int64_t)keys[k];
            lo = prev + 1, hi = cur;
            if (occ_bits && k < n && cur != prev) atomicOr(&occ_bits[cur >> 5], 1u << (cur & 31));
        }
        // short ranges (the common case: a few cells between neighbouring
        // points) by their own lane, long ones by the whole warp
        const bool longr = hi - lo >= 64;
        if (!longr)
            for (int64_t c = lo; c <= hi; ++c) cs[c] = (int32_t)k;
        unsigned todo = __ballot_sync(0xffffffffu, longr);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t l = __shfl_sync(0xffffffffu, lo, src), h = __shfl_sync(0xffffffffu, hi, src);
            const int32_t v = (int32_t)(w * 32 + src);
            for (int64_t c = l + lane; c <= h; c += 32) cs[c] = v;
        }
    }
}

// Source shard by key range (world > 1): a histogram of the top bits of the
// ordering keys (shared-memory privatised, 2^12 buckets), then the stable
// selection of the keys in a bucket range; sorting only the selection gives
// exactly the slice of the full stable sort (ties keep original-index order).
// shard bucket of an ordering key: the top key bits, or (dense grid, nx > 0)
// the cell's x index scaled to the bucket range, so a shard is an x-slab
// (every slab of a building-scale scene then holds floor, ceiling and boxes
// alike; z-slabs put the floor and the ceiling in two cheap shards)
__device__ __forceinline__ uint32_t shard_bucket(uint32_t k, int shift, int nx) {
    if (nx > 0) return (uint32_t)(((uint64_t)(k % (uint32_t)nx) * kShardBuckets) / (uint64_t)nx);
    return min(k >> shift, (uint32_t)kShardBuckets - 1u);
}
__global__ void k_key_hist(const uint32_t* __restrict__ keys, int64_t n, int shift, int nx,
                           const uint32_t* __restrict__ live, uint32_t* __restrict__ hist) {
    // hist[b] = points of bucket b, hist[kShardBuckets + b] = those whose
    // 27-cell stencil holds a target (dense grid: bit `key` of the dilated
    // occupancy bitmap; the live ones run the full search: the work estimate)
    __shared__ uint32_t h[2 * kShardBuckets];
    for (int t = threadIdx.x; t < 2 * kShardBuckets; t += blockDim.x) h[t] = 0u;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        const uint32_t b = shard_bucket(k, shift, nx);
        atomicAdd(&h[b], 1u);
        if (live && ((__ldg(&live[k >> 5]) >> (k & 31)) & 1u)) atomicAdd(&h[kShardBuckets + b], 1u);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * kShardBuckets; t += blockDim.x)
        if (h[t]) atomicAdd(&hist[t], h[t]);
}
__global__ void k_key_flags(const uint32_t* __restrict__ keys, int64_t n, int shift, int nx, uint32_t blo,
                            uint32_t bhi, uint8_t* __restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = shard_bucket(keys[i], shift, nx);
        flags[i] = (b >= blo && b <= bhi) ? 1 : 0;
    }
}

// hashed grid: occupancy of coarse cells (2^shift fine cells per axis), the
// live-query test's structure when no dense per-cell bitmap fits
__global__ void k_coarse_bits(const float4* __restrict__ tpos, int64_t n, GridDev g, int shift, int cnx, int cny,
                              uint32_t* __restrict__ bits) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 p = tpos[i];
        const int cx = min(max(cell_coord((double)p.x, g.ox, g.inv_h, g.nx), 0), g.nx - 1) >> shift;
        const int cy = min(max(cell_coord((double)p.y, g.oy, g.inv_h, g.ny), 0), g.ny - 1) >> shift;
        const int cz = min(max(cell_coord((double)p.z, g.oz, g.inv_h, g.nz), 0), g.nz - 1) >> shift;
        const int64_t k = ((int64_t)cz * cny + cy) * cnx + cx;
        atomicOr(&bits[k >> 5], 1u << (k & 31));
    }
}

// x-order inside cells (O3G_OPT_XSORT): key = cell << 32 | order-preserving
// bits of x, value = current position; then the target is permuted
__global__ void k_xkeys(const float4* __restrict__ tpos, int64_t n, GridDev g, uint64_t* __restrict__ keys,
                        int32_t* __restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 p = tpos[i];
        const int cx = min(max(cell_coord((double)p.x, g.ox, g.inv_h, g.nx), 0), g.nx - 1);
        const int cy = min(max(cell_coord((double)p.y, g.oy, g.inv_h, g.ny), 0), g.ny - 1);
        const int cz = min(max(cell_coord((double)p.z, g.oz, g.inv_h, g.nz), 0), g.nz - 1);
        uint32_t u = __float_as_uint(p.x);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        keys[i] = ((uint64_t)grid_index_dense(g, cx, cy, cz) << 32) | u;
        vals[i] = (int32_t)i;
    }
}
__global__ void k_permute_target(const float4* __restrict__ tpos, const float4* __restrict__ tnrm,
                                 const int32_t* __restrict__ perm, int64_t n, float4* __restrict__ opos,
                                 float4* __restrict__ onrm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = perm[i];
        opos[i] = tpos[v];
        onrm[i] = tnrm[v];
    }
}

// tile starts of the (sorted) source: a new tile where the brick id (key >>
// shift) changes (shift 32: never) and every `tq` queries inside a brick run.
// run_start[i] = the start of i's run (an inclusive max-scan of these marks)
__global__ void k_run_marks(const uint32_t* __restrict__ keys, int64_t n, int shift,
                            int32_t* __restrict__ mark) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool start = i == 0 || (shift < 32 && (keys[i] >> shift) != (keys[i - 1] >> shift));
        mark[i] = start ? (int32_t)i : 0;
    }
}
__global__ void k_tile_flags(const int32_t* __restrict__ run_start, int64_t n, int tq,
                             uint8_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        flag[i] = ((i - run_start[i]) % tq) == 0;
}

__global__ void k_histogram(const uint32_t* __restrict__ keys, int64_t n, int32_t* counts,
                            unsigned long long* occupied) {
    int occ = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        occ += atomicAdd(&counts[keys[i]], 1) == 0;   // first point of its cell
    if (occupied) {
        for (int o = 16; o; o >>= 1) occ += __shfl_xor_sync(0xffffffffu, occ, o);
        if ((threadIdx.x & 31) == 0 && occ) atomicAdd(occupied, (unsigned long long)occ);
    }
}

// Counting-sort placement of the target (a one-digit LSD radix sort with the
// cell index as the digit): cursor starts as a copy of cell_start; each point
// takes the next slot of its cell. Order inside a cell is arbitrary — every
// consumer breaks ties by the original index, so results do not depend on it.
__global__ void k_scatter_target(const float* __restrict__ xyz, const float* __restrict__ nrm,
                                 const uint32_t* __restrict__ keys, int64_t n, int32_t* cursor,
                                 float4* __restrict__ tpos, float4* __restrict__ tnrm) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t pos = atomicAdd(&cursor[keys[i]], 1);
        tpos[pos] = make_float4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], __int_as_float((int32_t)i));
        tnrm[pos] = nrm ? make_float4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], 0.f)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

__global__ void k_gather_target(const float* __restrict__ xyz, const float* __restrict__ nrm,
                                const int32_t* __restrict__ vals, const uint32_t* __restrict__ keys,
                                int64_t n, float4* __restrict__ tpos, float4* __restrict__ tnrm,
                                unsigned long long* occupied) {
    int occ = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = vals[i];
        tpos[i] = make_float4(xyz[3 * (int64_t)v], xyz[3 * (int64_t)v + 1], xyz[3 * (int64_t)v + 2],
                              __int_as_float(v));
        tnrm[i] = nrm ? make_float4(nrm[3 * (int64_t)v], nrm[3 * (int64_t)v + 1], nrm[3 * (int64_t)v + 2], 0.f)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
        occ += (i == 0 || keys[i] != keys[i - 1]);
    }
    for (int o = 16; o; o >>= 1) occ += __shfl_xor_sync(0xffffffffu, occ, o);
    if ((threadIdx.x & 31) == 0 && occ) atomicAdd(occupied, (unsigned long long)occ);
}

__global__ void k_gather_source(const float* __restrict__ xyz, const int32_t* __restrict__ vals,
                                int64_t lo, int64_t hi, float4* __restrict__ out) {
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = vals[i];
        out[i - lo] = make_float4(xyz[3 * (int64_t)v], xyz[3 * (int64_t)v + 1], xyz[3 * (int64_t)v + 2],
                                  __int_as_float(v));
    }
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void k_occupancy_bits(const int32_t* __restrict__ cs, int64_t ncells,
                                 uint32_t* __restrict__ bits) {
    const int64_t nw = (ncells + 31) / 32;
    for (int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; w < nw;
         w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t k = w * 32 + (threadIdx.x & 31);
        const bool occ = k < ncells && cs[k + 1] > cs[k];
        const uint32_t b = __ballot_sync(0xffffffffu, occ);
        if ((threadIdx.x & 31) == 0) bits[w] = b;
    }
}

// 32 bits of `in` starting at bit position `pos` (zeros outside [0, nbits))
__device__ __forceinline__ uint32_t bits_at(const uint32_t* in, int64_t nw, int64_t pos) {
    const int64_t wi = pos >= 0 ? pos / 32 : -((-pos + 31) / 32);
    const int sh = (int)(pos - wi * 32);
    const uint32_t lo = (wi >= 0 && wi < nw) ? in[wi] : 0u;
    const uint32_t hi = (wi + 1 >= 0 && wi + 1 < nw) ? in[wi + 1] : 0u;
    return __funnelshift_r(lo, hi, sh);
}

__global__ void k_dilate_bits(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                              int64_t nw, int64_t off) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw;
         w += (int64_t)gridDim.x * blockDim.x)
        out[w] = in[w] | bits_at(in, nw, w * 32 - off) | bits_at(in, nw, w * 32 + off);
}

static int blocks_for(int64_t n, int threads, int cap = 148 * 16) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    return (int)(b < cap ? b : cap);
}

void launch_bbox(const float* xyz, int64_t n, uint32_t* mm, int32_t* nonfinite, int sms,
                 cudaStream_t s) {
    k_bbox<<<blocks_for(n, 256, sms * 8), 256, 0, s>>>(xyz, n, mm, nonfinite);
}
void launch_check_finite(const float* v, int64_t count, int32_t* nonfinite, int sms,
                         cudaStream_t s) {
    k_check_finite<<<blocks_for(count, 256, sms * 8), 256, 0, s>>>(v, count, nonfinite);
}
void launch_cell_keys(const float* xyz, int64_t n, const GridDev& g, const double* T,
                      uint32_t* keys, int32_t* vals, cudaStream_t s, int brick) {
    static const double I[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
    const double* t = T ? T : I;
    k_cell_keys<<<blocks_for(n, 256), 256, 0, s>>>(xyz, n, g, T != nullptr, t[0], t[1], t[2], t[3],
                                                   t[4], t[5], t[6], t[7], t[8], t[9], t[10], t[11],
                                                   keys, vals, brick);
}
void launch_cs_runs(const uint32_t* keys, int64_t n, int32_t* runs, uint32_t* occ_bits, cudaStream_t s) {
    k_cs_runs<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, runs, occ_bits);
}
void launch_cs_fill(const uint32_t* keys, int64_t n, int64_t cells, int32_t* cs, uint32_t* occ_bits,
                    cudaStream_t s) {
    k_cs_fill<<<blocks_for(n / 32 + 1, 8), 256, 0, s>>>(keys, n, cells, cs, occ_bits);
}
void launch_key_hist(const uint32_t* keys, int64_t n, int shift, int nx, const uint32_t* live, uint32_t* hist,
                     int sms, cudaStream_t s) {
    cudaMemsetAsync(hist, 0, 2 * kShardBuckets * sizeof(uint32_t), s);
    k_key_hist<<<blocks_for(n, 256, sms * 2), 256, 0, s>>>(keys, n, shift, nx, live, hist);
}
void launch_key_flags(const uint32_t* keys, int64_t n, int shift, int nx, uint32_t blo, uint32_t bhi,
                      uint8_t* flags, cudaStream_t s) {
    k_key_flags<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, shift, nx, blo, bhi, flags);
}
void launch_coarse_bits(const float4* tpos, int64_t n, const GridDev& g, int shift, int cnx, int cny,
                        uint32_t* bits, cudaStream_t s) {
    k_coarse_bits<<<blocks_for(n, 256), 256, 0, s>>>(tpos, n, g, shift, cnx, cny, bits);
}
void launch_xkeys(const float4* tpos, int64_t n, const GridDev& g, uint64_t* keys, int32_t* vals,
                  cudaStream_t s) {
    k_xkeys<<<blocks_for(n, 256), 256, 0, s>>>(tpos, n, g, keys, vals);
}
void launch_permute_target(const float4* tpos, const float4* tnrm, const int32_t* perm, int64_t n,
                           float4* opos, float4* onrm, cudaStream_t s) {
    k_permute_target<<<blocks_for(n, 256), 256, 0, s>>>(tpos, tnrm, perm, n, opos, onrm);
}
void launch_run_marks(const uint32_t* keys, int64_t n, int shift, int32_t* mark, cudaStream_t s) {
    k_run_marks<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, shift, mark);
}
void launch_tile_flags(const int32_t* run_start, int64_t n, int tq, uint8_t* flag, cudaStream_t s) {
    k_tile_flags<<<blocks_for(n, 256), 256, 0, s>>>(run_start, n, tq, flag);
}
void launch_histogram(const uint32_t* keys, int64_t n, int32_t* counts, unsigned long long* occupied,
                      cudaStream_t s) {
    k_histogram<<<blocks_for(n, 256), 256, 0, s>>>(keys, n, counts, occupied);
}
void launch_scatter_target(const float* xyz, const float* nrm, const uint32_t* keys, int64_t n,
                           int32_t* cursor, float4* tpos, float4* tnrm, cudaStream_t s) {
    k_scatter_target<<<blocks_for(n, 256), 256, 0, s>>>(xyz, nrm, keys, n, cursor, tpos, tnrm);
}
void launch_gather_target(const float* xyz, const float* nrm, const int32_t* vals,
                          const uint32_t* keys, int64_t n, float4* tpos, float4* tnrm,
                          unsigned long long* occupied, cudaStream_t s) {
    k_gather_target<<<blocks_for(n, 256), 256, 0, s>>>(xyz, nrm, vals, keys, n, tpos, tnrm, occupied);
}
void launch_gather_source(const float* xyz, const int32_t* vals, int64_t lo, int64_t hi,
                          float4* out, cudaStream_t s) {
    k_gather_source<<<blocks_for(hi - lo, 256), 256, 0, s>>>(xyz, vals, lo, hi, out);
}
void launch_dilate3(uint32_t* bits, uint32_t* tmp, int64_t ncells, int64_t nx, int64_t nxny, cudaStream_t s) {
    const int64_t nw = (ncells + 31) / 32;
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(bits, tmp, nw, 1);
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(tmp, bits, nw, nx);
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(bits, tmp, nw, nxny);
    cudaMemcpyAsync(bits, tmp, nw * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
}
void launch_nbr_bits(const int32_t* cs, int64_t ncells, int64_t nx, int64_t nxny, uint32_t* tmp,
                     uint32_t* out, cudaStream_t s) {
    const int64_t nw = (ncells + 31) / 32;
    k_occupancy_bits<<<blocks_for(nw * 32, 256), 256, 0, s>>>(cs, ncells, out);
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(out, tmp, nw, 1);
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(tmp, out, nw, nx);
    k_dilate_bits<<<blocks_for(nw, 256), 256, 0, s>>>(out, tmp, nw, nxny);
    cudaMemcpyAsync(out, tmp, nw * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s);
}

void launch_fill_i32(int32_t* p, int64_t n, int32_t v, cudaStream_t s) {
    k_fill_i32<<<blocks_for(n, 256), 256, 0, s>>>(p, n, v);
}

// every 32-byte certificate record's first half := {-1, all ones, 0, 0}
// (no winner, invalid certificate); the second half is left as it is
__global__ void k_cert_reset(float4* cert, int64_t n, const IcpState* st) {
    if (!st->creset) return;   // (records of earlier runs are already invalid by their pass tag)
    const float4 v = make_float4(__int_as_float(-1), __int_as_float(-1), 0.f, 0.f);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        cert[2 * i] = v;
}
void launch_cert_reset(float4* cert, int64_t n, const IcpState* st, cudaStream_t s) {
    k_cert_reset<<<blocks_for(n, 256), 256, 0, s>>>(cert, n, st);
}

}  // namespace o3g
