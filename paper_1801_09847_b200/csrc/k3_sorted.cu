// k3_sorted.cu — K3 variant 3 (O3G_OPT_SEARCH=3; measured slower than the default variant 1): the correspondence + reduction pass
// organised around a per-block tile of 128 spatially consecutive queries.
//
// Same contract and bit-identical correspondences as k3_corr_reduce
// (DESIGN.md §5.3). Why the reorganisation: on surface scenes the number of
// candidates per query is strongly bimodal (about half the queries of the
// 16M config have none at T_init, p99 is ~5x the mean), so a warp that holds
// 32 consecutive queries waits for its longest list. Here
//   S  each thread sets up one query of the tile (s' = T s in fp64, cell,
//      the 9 x-row ranges from the dense cell table) into shared memory;
//   R  the tile is stably sorted by candidate count (6-bit LSD radix sort,
//      ballot + popc per pass), so each warp gets queries of similar length;
//   P  each thread runs the branch-free fp32 pass over its (sorted) query's
//      candidates, the exact fp64 decision (rare exact rescan on near-ties),
//      and the warp accumulates its 32 records with fp64 tensor-core MMAs
//      (V^T W, see k3_balanced).
// Everything is deterministic: the sort is stable and every sum has a fixed
// order.
#include "k3_common.cuh"

namespace o3g {

constexpr int kT3 = 128;
constexpr int kT3W = kT3 / 32;

template <bool WRITE_CORR, bool HASHED>
__global__ void __launch_bounds__(kT3, 8) k3_sorted(const K3Args a) {
    constexpr int S = HASHED ? 18 : 9;
    __shared__ double sT[12];
    __shared__ double qd[4][kT3];          // s'x, s'y, s'z, E1
    __shared__ float4 qf[kT3];             // fl32(s'), thr(r^2)
    __shared__ int2 segs[S][kT3];          // non-empty x-row ranges [b, e)
    __shared__ int qn[kT3];                // nseg | count << 5
    __shared__ int qi[kT3];                // original source index
    __shared__ short pslot[2][kT3];        // radix-sort ping-pong: slot at position
    __shared__ unsigned char pkey[2][kT3];
    __shared__ int wz[2][kT3W];
    __shared__ double vw[kT3W][9 * kVW];   // per-warp record staging
    __shared__ double red[kT3W][64];

    if (a.st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 12) sT[tid] = a.st->T[tid];
    __syncthreads();

    const GridDev g = a.g;
    const double r2 = a.r2;
    double acc0 = 0.0, acc1 = 0.0;
    const int ntiles = (a.n + kT3 - 1) / kT3;

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // ------------------------------------------------ S: query setup
        {
            const int i = tile * kT3 + tid;
            int nseg = 0, c = 0, oidx = -1;
            if (i < a.n) {
                const float4 p = __ldg(&a.src[i]);
                oidx = __float_as_int(p.w);
                double sx, sy, sz;
                xform_rn(sT, p.x, p.y, p.z, sx, sy, sz);
                const int cx = cell_coord(sx, g.ox, g.inv_h, g.nx);
                const int cy = cell_coord(sy, g.oy, g.inv_h, g.ny);
                const int cz = cell_coord(sz, g.oz, g.inv_h, g.nz);
                const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
                const int ylo = max(cy - 1, 0), yhi = min(cy + 1, g.ny - 1);
                const int zlo = max(cz - 1, 0), zhi = min(cz + 1, g.nz - 1);
                if (!HASHED) {
                    if (xlo <= xhi) {
                        // row (y, z) window [xlo, xhi] = cell_start[row + xlo .. row + xhi + 1]
                        const int w = xhi - xlo + 1;
                        const long long sy_ = g.nx, sz_ = (long long)g.nx * g.ny;
                        const int* p0 = a.cell_start + ((long long)(cz - 1) * g.ny + (cy - 1)) * g.nx + xlo;
                        int bb[9], ee[9];
#pragma unroll
                        for (int r = 0; r < 9; ++r) {
                            const int z = cz + r / 3 - 1, y = cy + r % 3 - 1;
                            const bool ok = z >= zlo && z <= zhi && y >= ylo && y <= yhi;
                            const int* pr = p0 + (r / 3) * sz_ + (r % 3) * sy_;
                            bb[r] = ok ? __ldg(pr) : 0;
                            ee[r] = ok ? __ldg(pr + w) : 0;
                        }
#pragma unroll
                        for (int r = 0; r < 9; ++r) {
                            if (ee[r] > bb[r]) {
                                segs[nseg][tid] = make_int2(bb[r], ee[r]);
                                ++nseg;
                                c += ee[r] - bb[r];
                            }
                        }
                    }
                } else if (xlo <= xhi && ylo <= yhi && zlo <= zhi) {
                    for (int z = zlo; z <= zhi; ++z) {
                        for (int y = ylo; y <= yhi; ++y) {
                            const uint32_t s0 = (grid_row_hash(y, z) + (uint32_t)xlo) & g.hmask;
                            const uint32_t cnt = (uint32_t)(xhi - xlo + 1);
                            int b0 = __ldg(&a.cell_start[s0]), e0, b1 = 0, e1 = 0;
                            if ((uint64_t)s0 + cnt <= (uint64_t)g.hmask + 1) {
                                e0 = __ldg(&a.cell_start[s0 + cnt]);
                            } else {
                                e0 = __ldg(&a.cell_start[(int64_t)g.hmask + 1]);
                                b1 = __ldg(&a.cell_start[0]);
                                e1 = __ldg(&a.cell_start[(s0 + cnt) & g.hmask]);
                            }
                            if (e0 > b0) { segs[nseg][tid] = make_int2(b0, e0); ++nseg; c += e0 - b0; }
                            if (e1 > b1) { segs[nseg][tid] = make_int2(b1, e1); ++nseg; c += e1 - b1; }
                        }
                    }
                }
                float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                double E1 = 0.0;
                if (c > 0) {
                    f.x = __double2float_rn(sx);
                    f.y = __double2float_rn(sy);
                    f.z = __double2float_rn(sz);
                    E1 = (fabs(sx - (double)f.x) + fabs(sy - (double)f.y) + fabs(sz - (double)f.z)) *
                         (1.0 + 9.5367431640625e-07);
                    f.w = prefilter_thr(r2, E1, a.dmax, a.inv_dmax);
                }
                qd[0][tid] = sx, qd[1][tid] = sy, qd[2][tid] = sz, qd[3][tid] = E1;
                qf[tid] = f;
            }
            qn[tid] = nseg | (c << 5);
            qi[tid] = oidx;
            pslot[0][tid] = (short)tid;
            pkey[0][tid] = (unsigned char)(63 - min(c, 63));   // ascending key = descending count
        }
        __syncthreads();

        // ------------------------------------ R: stable radix sort by key
        int cur = 0;
#pragma unroll 1
        for (int bit = 0; bit < 6; ++bit) {
            const int slot = pslot[cur][tid];
            const int key = pkey[cur][tid];
            const bool one = (key >> bit) & 1;
            const unsigned zb = __ballot_sync(0xffffffffu, !one);
            if (lane == 0) wz[bit & 1][warp] = __popc(zb);
            __syncthreads();
            int zbefore = 0, ztot = 0;
#pragma unroll
            for (int w = 0; w < kT3W; ++w) {
                const int z = wz[bit & 1][w];
                ztot += z;
                zbefore += w < warp ? z : 0;
            }
            const unsigned below = (1u << lane) - 1u;
            const int pos = one ? ztot + (warp * 32 - zbefore) + __popc(~zb & below)
                                : zbefore + __popc(zb & below);
            pslot[cur ^ 1][pos] = (short)slot;
            pkey[cur ^ 1][pos] = (unsigned char)key;
            cur ^= 1;
            __syncthreads();
        }

        // ----------------------- P: pass 1, decision, accumulation (sorted)
        const int q = pslot[cur][tid];
        const int qn_ = qn[q], nseg = qn_ & 31, c = qn_ >> 5;
        int win = -1, widx = -1;
        double wd2 = 0.0, sx = 0.0, sy = 0.0, sz = 0.0;
        float4 wq = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c > 0) {
            const float4 f = qf[q];
            float m1 = CUDART_INF_F, m2 = CUDART_INF_F;
            int j1 = -1;
            {
                int k = 0;
                int2 sg = segs[0][q];
                int j = sg.x, e = sg.y;
                for (int it = 0; it < c; ++it) {
                    if (j == e) {
                        ++k;
                        sg = segs[k][q];
                        j = sg.x, e = sg.y;
                    }
                    const float4 t = __ldg(&a.tpos[j]);
                    const float ux = t.x - f.x, uy = t.y - f.y, uz = t.z - f.z;
                    const float df = fmaf(uz, uz, fmaf(uy, uy, ux * ux));
                    const bool lt = df < m1;
                    m2 = fminf(m2, lt ? m1 : df);
                    m1 = lt ? df : m1;
                    j1 = lt ? j : j1;
                    ++j;
                }
            }
            if (m1 <= f.w) {
                sx = qd[0][q], sy = qd[1][q], sz = qd[2][q];
                const double E1 = qd[3][q];
                const float4 t = __ldg(&a.tpos[j1]);
                const double dx = __dsub_rn(sx, (double)t.x), dy = __dsub_rn(sy, (double)t.y),
                             dz = __dsub_rn(sz, (double)t.z);
                const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
                const double B = d2 <= r2 ? d2 : r2;
                if (m2 > prefilter_thr(B, E1, a.dmax, a.inv_dmax)) {
                    if (d2 <= r2) win = j1, widx = __float_as_int(t.w), wd2 = d2, wq = t;
                } else {
                    // near-tie (or a point visited twice): exact filtered rescan
                    double bd = CUDART_INF;
                    int bidx = INT_MAX;
                    float thr = f.w;
                    for (int k = 0; k < nseg; ++k) {
                        const int2 sg = segs[k][q];
                        for (int j = sg.x; j < sg.y; ++j) {
                            const float4 u = __ldg(&a.tpos[j]);
                            const float ux = u.x - f.x, uy = u.y - f.y, uz = u.z - f.z;
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
        }
        if (WRITE_CORR) {
            const int oi = qi[q];
            if (oi >= 0) a.corr_out[oi] = widx;
        }

        // A5/A6: records -> V (J, r, m) and W (J, m, d2); C += V^T W on the DMMA pipe
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
            double* st = vw[warp];
#pragma unroll
            for (int r = 0; r < 8; ++r) st[r * kVW + lane] = v[r];
            st[8 * kVW + lane] = d2w;
            __syncwarp();
            const int row = lane >> 2, kk = lane & 3, wrow = row < 6 ? row : row + 1;
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
                if ((matched >> (4 * c4)) & 0xFu)
                    dmma884(acc0, acc1, st[row * kVW + 4 * c4 + kk], st[wrow * kVW + 4 * c4 + kk]);
            }
            __syncwarp();
        }
        __syncthreads();   // the next tile reuses every shared array
    }

    red[warp][(lane >> 2) * 8 + 2 * (lane & 3)] = acc0;
    red[warp][(lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc1;
    __syncthreads();
    if (tid < kTermStride) {
        double s = 0.0;
        if (tid < kTerms) {
            const int ci = term_cidx(tid);
            for (int w = 0; w < kT3W; ++w) s += red[w][ci];
        }
        a.block_partials[(size_t)blockIdx.x * kTermStride + tid] = s;
    }
}

template <bool W, bool H>
static int occ3() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_sorted<W, H>, kT3, 0);
    return b;
}

int k3_sorted_blocks_per_sm(bool write_corr, int hashed) {
    if (hashed) return write_corr ? occ3<true, true>() : occ3<false, true>();
    return write_corr ? occ3<true, false>() : occ3<false, false>();
}

void launch_k3_sorted(const K3Args& a, int blocks, bool write_corr, cudaStream_t s) {
    if (a.g.hashed) {
        if (write_corr) k3_sorted<true, true><<<blocks, kT3, 0, s>>>(a);
        else k3_sorted<false, true><<<blocks, kT3, 0, s>>>(a);
    } else {
        if (write_corr) k3_sorted<true, false><<<blocks, kT3, 0, s>>>(a);
        else k3_sorted<false, false><<<blocks, kT3, 0, s>>>(a);
    }
}

}  // namespace o3g
