// k3_tiled.cu — K3 variant 4: the correspondence + reduction pass with the
// target neighbourhood of a whole query tile staged in shared memory.
//
// Same contract and bit-identical correspondences as k3_corr_reduce /
// k3_balanced; dense cell table only (the host maps a
// hashed grid to variant 1). Why: k3_balanced is bound by the latency of its
// per-lane gathers (L2 round trips through the 18 row-boundary loads and the
// candidate loads; long-scoreboard ~50% of stalls) and by L1 wavefronts.
// The source is ordered by 8^3-cell bricks (Morton) and cut into tiles of at
// most 256 queries that never straddle a brick (o3g_set_source), so a tile's
// queries stay spatially compact under any rigid motion. Per tile:
//   A  every thread transforms 2 queries (fp64), finds their cells and the
//      live ones (dilated occupancy bitmap); the live queries are compacted
//      in tile order and their cell bounding box is reduced;
//   B  the box grown by one cell is the tile's halo: its x-row boundaries are
//      read from the dense table with coalesced row loads, scanned into a
//      local cell table, and every target point of the halo is copied into
//      shared memory row by row (coalesced float4 loads);
//   D  warps take 32 live queries at a time and run the k3_balanced search
//      (9 x-rows, branch-free fp32 pass, exact fp64 decision / rescan) on the
//      staged copy, then accumulate their records on the fp64 tensor cores.
// A tile whose halo exceeds the staging capacity runs phase D on global
// memory (the k3_balanced path), so any input is handled.
#include "k3_common.cuh"

namespace o3g {

constexpr int kTT = 128;           // threads per block
constexpr int kTWarps = kTT / 32;
constexpr int kTQ = kTileQ;        // queries per tile (max; one per thread in phase A)
constexpr int kTMaxP = 1024;       // staged target points (16 KB)
constexpr int kTMaxE = 2048;       // local cell-table entries
constexpr int kTMaxR = 256;        // halo x-rows
static_assert(kTMaxR == 2 * kTT && kTQ == kTT, "phase A: one query per thread; row scan: two rows");
constexpr size_t kTWarpBytes = 9 * kVW * sizeof(double);   // >= 9 * 32 * sizeof(int2)
constexpr size_t kTDynSmem = kTMaxP * sizeof(float4) + kTWarps * kTWarpBytes;

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// exclusive block scan of one int per thread; returns the total
__device__ __forceinline__ int tile_scan(int v, int* wsum, int& excl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kTWarps; ++w) {
        const int t = wsum[w];
        before += w < warp ? t : 0;
        total += t;
    }
    __syncthreads();
    excl = before + x - v;
    return total;
}

template <bool WRITE_CORR>
__global__ void __launch_bounds__(kTT, 6) k3_tiled(const K3Args a) {
    extern __shared__ __align__(16) unsigned char tsm[];
    float4* tile = (float4*)tsm;
    __shared__ double sT[12];
    __shared__ int lcs[kTMaxE];        // local cell starts, row-major over the halo rows
    __shared__ int gofs[kTMaxR];       // global index = local index + gofs[row]
    __shared__ int qlist[kTQ];         // live queries of the tile (offsets, tile order)
    __shared__ int s_box[6];           // min cx, cy, cz, max cx, cy, cz of live queries
    __shared__ int wsum[kTWarps];
    __shared__ int s_info[2];          // live count, staged flag

    if (a.st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 12) sT[tid] = a.st->T[tid];
    const GridDev g = a.g;
    const double r2 = a.r2;
    const int* __restrict__ cs = a.cell_start;
    int2* segs = (int2*)(tsm + kTMaxP * sizeof(float4) + (size_t)warp * kTWarpBytes);
    double* vw = (double*)segs;
    double acc0 = 0.0, acc1 = 0.0;
    __syncthreads();

    for (int tile_i = blockIdx.x; tile_i < a.ntiles; tile_i += gridDim.x) {
        const int q0 = a.tiles[tile_i];
        const int qend = tile_i + 1 < a.ntiles ? a.tiles[tile_i + 1] : a.n;
        // ------------------------------------------------ A: live queries
        if (tid < 3) s_box[tid] = INT_MAX, s_box[3 + tid] = INT_MIN;
        __syncthreads();
        int L = 0;
        {
            const int qo = tid, i = q0 + qo;
            bool live = false;
            int cx = 0, cy = 0, cz = 0;
            if (i < qend) {
                const float4 p = __ldg(&a.src[i]);
                double sx, sy, sz;
                xform_rn(sT, p.x, p.y, p.z, sx, sy, sz);
                cx = cell_coord(sx, g.ox, g.inv_h, g.nx);
                cy = cell_coord(sy, g.oy, g.inv_h, g.ny);
                cz = cell_coord(sz, g.oz, g.inv_h, g.nz);
                if (cx >= -1 && cx <= g.nx && cy >= -1 && cy <= g.ny && cz >= -1 && cz <= g.nz) {
                    const int kc = (min(max(cz, 0), g.nz - 1) * g.ny + min(max(cy, 0), g.ny - 1)) * g.nx +
                                   min(max(cx, 0), g.nx - 1);
                    live = a.nbr_bits && !g.hashed ? ((__ldg(&a.nbr_bits[kc >> 5]) >> (kc & 31)) & 1u) : true;
                }
                if (WRITE_CORR && !live) a.corr_out[__float_as_int(p.w)] = -1;
            }
            int excl;
            const int tot = tile_scan(live ? 1 : 0, wsum, excl);
            if (live) qlist[L + excl] = qo;
            L += tot;
            const int mnx = __reduce_min_sync(0xffffffffu, live ? cx : INT_MAX);
            const int mny = __reduce_min_sync(0xffffffffu, live ? cy : INT_MAX);
            const int mnz = __reduce_min_sync(0xffffffffu, live ? cz : INT_MAX);
            const int mxx = __reduce_max_sync(0xffffffffu, live ? cx : INT_MIN);
            const int mxy = __reduce_max_sync(0xffffffffu, live ? cy : INT_MIN);
            const int mxz = __reduce_max_sync(0xffffffffu, live ? cz : INT_MIN);
            if (lane == 0 && mxx != INT_MIN) {
                atomicMin(&s_box[0], mnx), atomicMin(&s_box[1], mny), atomicMin(&s_box[2], mnz);
                atomicMax(&s_box[3], mxx), atomicMax(&s_box[4], mxy), atomicMax(&s_box[5], mxz);
            }
        }
        __syncthreads();
        if (L == 0) continue;   // block-uniform

        // ------------------------------------------------ B: stage the halo
        const int x0 = max(s_box[0] - 1, 0), x1 = min(s_box[3] + 1, g.nx - 1);
        const int y0 = max(s_box[1] - 1, 0), y1 = min(s_box[4] + 1, g.ny - 1);
        const int z0 = max(s_box[2] - 1, 0), z1 = min(s_box[5] + 1, g.nz - 1);
        const int hx = x1 - x0 + 1, hy = y1 - y0 + 1, hz = z1 - z0 + 1;
        const int W = hx + 1;                       // entries per row: starts of x0..x1, end
        const long long nrows_l = (long long)hy * hz;
        bool staged = x0 <= x1 && y0 <= y1 && z0 <= z1 && nrows_l <= kTMaxR && nrows_l * W <= kTMaxE;
        const int nrows = staged ? (int)nrows_l : 0;
        if (staged) {
            // asynchronous copies (no register staging): every load of the
            // tile is in flight at once
            for (int e = tid; e < nrows * W; e += kTT) {
                const int r = e / W, u = e - r * W;
                const int z = z0 + r / hy, y = y0 + r % hy;
                cp_async4(&lcs[e], &cs[(z * g.ny + y) * g.nx + x0 + u]);
            }
            cp_async_wait_all();
            __syncthreads();
            int ex0, ex1;
            // row lengths -> local row starts (kTMaxR = 2 kTT rows: two scans)
            const int v0 = tid < nrows ? lcs[tid * W + hx] - lcs[tid * W] : 0;
            const int t0 = tile_scan(v0, wsum, ex0);
            const int v1 = tid + kTT < nrows ? lcs[(tid + kTT) * W + hx] - lcs[(tid + kTT) * W] : 0;
            const int t1 = tile_scan(v1, wsum, ex1);
            staged = t0 + t1 <= kTMaxP;   // block-uniform
            if (staged) {
                if (tid < nrows) gofs[tid] = lcs[tid * W] - ex0;
                if (tid + kTT < nrows) gofs[tid + kTT] = lcs[(tid + kTT) * W] - (t0 + ex1);
                __syncthreads();
                for (int e = tid; e < nrows * W; e += kTT) lcs[e] -= gofs[e / W];
                __syncthreads();
                for (int r = warp; r < nrows; r += kTWarps) {
                    const int lb = lcs[r * W], le = lcs[r * W + hx], gb = lb + gofs[r];
                    for (int k = lane; k < le - lb; k += 32) cp_async16(&tile[lb + k], &a.tpos[gb + k]);
                }
                cp_async_wait_all();
            }
            __syncthreads();
        }
        const float4* __restrict__ TP = staged ? tile : a.tpos;

        // ------------------------------------------------ D: search + accumulate
        for (int b = warp; b * 32 < L; b += kTWarps) {
            const int qi = b * 32 + lane;
            const int i = qi < L ? q0 + qlist[qi] : a.n;
            double sx = 0.0, sy = 0.0, sz = 0.0, E1 = 0.0;
            float shx = 0.f, shy = 0.f, shz = 0.f, thr0 = 0.f;
            int nseg = 0, c = 0;
            float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
            if (i < a.n) {
                p = __ldg(&a.src[i]);
                xform_rn(sT, p.x, p.y, p.z, sx, sy, sz);
                const int cx = cell_coord(sx, g.ox, g.inv_h, g.nx);
                const int cy = cell_coord(sy, g.oy, g.inv_h, g.ny);
                const int cz = cell_coord(sz, g.oz, g.inv_h, g.nz);
                const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
                const int ylo = max(cy - 1, 0), yhi = min(cy + 1, g.ny - 1);
                const int zlo = max(cz - 1, 0), zhi = min(cz + 1, g.nz - 1);
                if (xlo <= xhi) {
                    int bb[9], ee[9];
                    if (staged) {
                        // the halo contains the stencil of every live query of the tile
#pragma unroll
                        for (int r = 0; r < 9; ++r) {
                            const int z = cz + r / 3 - 1, y = cy + r % 3 - 1;
                            const bool ok = z >= zlo && z <= zhi && y >= ylo && y <= yhi;
                            const int base = ((z - z0) * hy + (y - y0)) * W - x0;
                            bb[r] = ok ? lcs[base + xlo] : 0;
                            ee[r] = ok ? lcs[base + xhi + 1] : 0;
                        }
                    } else {
                        const int w = xhi - xlo + 1;
                        const int rb0 = ((cz - 1) * g.ny + (cy - 1)) * g.nx + xlo;
#pragma unroll
                        for (int r = 0; r < 9; ++r) {
                            const int z = cz + r / 3 - 1, y = cy + r % 3 - 1;
                            const bool ok = z >= zlo && z <= zhi && y >= ylo && y <= yhi;
                            const int rb = rb0 + (r / 3) * g.nx * g.ny + (r % 3) * g.nx;
                            bb[r] = ok ? __ldg(cs + rb) : 0;
                            ee[r] = ok ? __ldg(cs + rb + w) : 0;
                        }
                    }
#pragma unroll
                    for (int r = 0; r < 9; ++r) {
                        if (ee[r] > bb[r]) {
                            segs[nseg * 32 + lane] = make_int2(bb[r], ee[r]);
                            ++nseg;
                            c += ee[r] - bb[r];
                        }
                    }
                }
                if (c > 0) {
                    shx = __double2float_rn(sx);
                    shy = __double2float_rn(sy);
                    shz = __double2float_rn(sz);
                    E1 = (fabs(sx - (double)shx) + fabs(sy - (double)shy) + fabs(sz - (double)shz)) *
                         (1.0 + 9.5367431640625e-07);
                    thr0 = prefilter_thr(r2, E1, a.dmax, a.inv_dmax);
                }
            }

            // pass 1: branch-free fp32 scan (m1 at j1, m2 over all others)
            float m1 = CUDART_INF_F, m2 = CUDART_INF_F;
            int j1 = -1;
            {
                const int2* sp = segs + lane;
                int2 sg = c > 0 ? *sp : make_int2(0, 0);
                int j = sg.x, e = sg.y;
                const float2 nsh = make_float2(-shx, -shy);
#pragma unroll 4
                for (int it = 0; it < c; ++it) {
                    if (j == e) {
                        sp += 32;
                        sg = *sp;
                        j = sg.x, e = sg.y;
                    }
                    const float4 t = TP[j];
                    const float2 uxy = __fadd2_rn(make_float2(t.x, t.y), nsh);
                    const float2 sq = __fmul2_rn(uxy, uxy);
                    const float uz = t.z - shz;
                    const float df = fmaf(uz, uz, __fadd_rn(sq.x, sq.y));
                    const bool lt = df < m1;
                    m2 = fminf(m2, lt ? m1 : df);
                    m1 = lt ? df : m1;
                    j1 = lt ? j : j1;
                    ++j;
                }
            }

            // decision (exact fp64 rule, R1-R3); win is an index into TP
            int win = -1, widx = -1;
            double wd2 = 0.0;
            float4 wq = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c > 0 && m1 <= thr0) {
                const float4 t = TP[j1];
                const double dx = __dsub_rn(sx, (double)t.x), dy = __dsub_rn(sy, (double)t.y),
                             dz = __dsub_rn(sz, (double)t.z);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                const double B = d2 <= r2 ? d2 : r2;
                if (m2 > prefilter_thr(B, E1, a.dmax, a.inv_dmax)) {
                    if (d2 <= r2) win = j1, widx = __float_as_int(t.w), wd2 = d2, wq = t;
                } else {
                    double bd = CUDART_INF;
                    int bidx = INT_MAX;
                    float thr = thr0;
                    for (int k = 0; k < nseg; ++k) {
                        const int2 sg = segs[k * 32 + lane];
                        for (int j = sg.x; j < sg.y; ++j) {
                            const float4 u = TP[j];
                            const float ux = u.x - shx, uy = u.y - shy, uz = u.z - shz;
                            if (fmaf(uz, uz, fmaf(uy, uy, ux * ux)) > thr) continue;
                            const double ex = __dsub_rn(sx, (double)u.x), ey = __dsub_rn(sy, (double)u.y),
                                         ez = __dsub_rn(sz, (double)u.z);
                            const double e2 = __dadd_rn(__dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey)),
                                                        __dmul_rn(ez, ez));
                            const int idx = __float_as_int(u.w);
                            if (e2 <= r2 && (e2 < bd || (e2 == bd && idx < bidx))) {
                                bd = e2, bidx = idx, win = j, wq = u;
                                thr = prefilter_thr(bd, E1, a.dmax, a.inv_dmax);
                            }
                        }
                    }
                    if (win >= 0) widx = bidx, wd2 = bd;
                }
            }
            if (staged && win >= 0) {
                // local -> global target index: the halo row holding win
                int lo = 0, hi = nrows - 1;
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (lcs[mid * W] <= win) lo = mid;
                    else hi = mid - 1;
                }
                win += gofs[lo];
            }
            if (WRITE_CORR && i < a.n) a.corr_out[__float_as_int(p.w)] = widx;

            // A5/A6: V = (J, r, m), W = (J, m, d2); C += V^T W on the DMMA pipe
            const unsigned matched = __ballot_sync(0xffffffffu, win >= 0);
            if (matched) {
                double v[8] = {0, 0, 0, 0, 0, 0, 0, 0}, d2w = 0.0;
                if (win >= 0) {
                    const float4 nf = __ldg(&a.tnrm[win]);
                    const double nx = nf.x, ny = nf.y, nz = nf.z;
                    v[0] = sy * nz - sz * ny;
                    v[1] = sz * nx - sx * nz;
                    v[2] = sx * ny - sy * nx;
                    v[3] = nx, v[4] = ny, v[5] = nz;
                    v[6] = (sx - (double)wq.x) * nx + (sy - (double)wq.y) * ny + (sz - (double)wq.z) * nz;
                    v[7] = 1.0;
                    d2w = wd2;
                }
                __syncwarp();
#pragma unroll
                for (int r = 0; r < 8; ++r) vw[r * kVW + lane] = v[r];
                vw[8 * kVW + lane] = d2w;
                __syncwarp();
                const int row = lane >> 2, kk = lane & 3, wrow = row < 6 ? row : row + 1;
#pragma unroll
                for (int c4 = 0; c4 < 8; ++c4) {
                    if ((matched >> (4 * c4)) & 0xFu)
                        dmma884(acc0, acc1, vw[row * kVW + 4 * c4 + kk], vw[wrow * kVW + 4 * c4 + kk]);
                }
            }
            __syncwarp();
        }
        __syncthreads();   // the next tile reuses every shared array
    }

    vw[(lane >> 2) * 8 + 2 * (lane & 3)] = acc0;   // C of this warp, on its own staging bytes
    vw[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc1;
    __syncthreads();
    if (tid < kTermStride) {
        double s = 0.0;
        if (tid < kTerms) {
            const int ci = term_cidx(tid);
            for (int w = 0; w < kTWarps; ++w)
                s += ((const double*)(tsm + kTMaxP * sizeof(float4) + (size_t)w * kTWarpBytes))[ci];
        }
        a.block_partials[(size_t)blockIdx.x * kTermStride + tid] = s;
    }
}

template <bool W>
static int occ4() {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k3_tiled<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTDynSmem);
        attr = true;
    }
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_tiled<W>, kTT, kTDynSmem);
    return b;
}

int k3_tiled_blocks_per_sm(bool write_corr) { return write_corr ? occ4<true>() : occ4<false>(); }

void launch_k3_tiled(const K3Args& a, int blocks, bool write_corr, cudaStream_t s) {
    occ4<true>(), occ4<false>();
    if (write_corr) k3_tiled<true><<<blocks, kTT, kTDynSmem, s>>>(a);
    else k3_tiled<false><<<blocks, kTT, kTDynSmem, s>>>(a);
}

}  // namespace o3g
