// icp_kernels.cu — the per-iteration hot path.
//
// K3 k3_corr_reduce: one thread per transformed source point (grid-stride
//   over the spatially sorted shard): s' = T s (A3), 27-cell fixed-radius
//   1-NN over the voxel-hash grid as 9 x-row ranges of the sorted target
//   (A4), point-to-plane residual + Jacobian accumulated in 29 fp64
//   registers (A5), then warp-shuffle -> block reduction to one 29-term
//   partial per block (A6). No atomics: every sum has a fixed order.
// K4 k_tail: fixed-order sum of the block partials (and, multi-GPU, of the
//   rank partials in rank order), then fitness / rmse / criteria, the 6x6
//   LDL^T solve, the SE(3) exponential and T <- exp(xi^) T (A8).
#include <float.h>
#include <math_constants.h>

#include "o3g_internal.cuh"

namespace o3g {

// ------------------------------------------------------------------- K3
// Prefilter threshold. For a query s' (fp64) let
// sh = fl32(s') and E1 >= ||s' - sh||_1 (1 + 2^-20). Every candidate whose
// exact fp64 distance d2_64 <= B satisfies
//   df = fl32(|t - sh|^2) <= (1+2^-20) (B (1+2^-20) + E1 (B/dmax + dmax) + E1^2)
// (AM-GM bounds 2 sqrt(B) by B/dmax + dmax), so rejecting df > thr never
// drops a candidate that could win or tie under the exact fp64 rule.
__device__ __forceinline__ float prefilter_thr(double B, double E1, double dmax, double inv_dmax) {
    const double k = 1.0 + 9.5367431640625e-07;  // 1 + 2^-20
    double v = B * k + E1 * (B * inv_dmax + dmax) + E1 * E1;
    return __double2float_ru(v * k);
}

template <bool PREFILTER, bool WRITE_CORR>
__global__ void __launch_bounds__(kK3Threads) k3_corr_reduce(const K3Args a) {
    __shared__ double sT[12];
    __shared__ double red[kK3Threads / 32][kTerms];
    if (a.st->done) return;  // the loop has stopped: uniform early exit
    if (threadIdx.x < 12) sT[threadIdx.x] = a.st->T[threadIdx.x];
    __syncthreads();

    double acc[kTerms];
#pragma unroll
    for (int k = 0; k < kTerms; ++k) acc[k] = 0.0;

    const GridDev g = a.g;
    const double r2 = a.r2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        const float4 p = __ldg(&a.src[i]);
        double sx, sy, sz;
        xform_rn(sT, p.x, p.y, p.z, sx, sy, sz);
        const int cx = cell_coord(sx, g.ox, g.inv_h, g.nx);
        const int cy = cell_coord(sy, g.oy, g.inv_h, g.ny);
        const int cz = cell_coord(sz, g.oz, g.inv_h, g.nz);
        const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
        const int ylo = max(cy - 1, 0), yhi = min(cy + 1, g.ny - 1);
        const int zlo = max(cz - 1, 0), zhi = min(cz + 1, g.nz - 1);

        double best_d2 = CUDART_INF;
        int best_j = -1, best_idx = INT_MAX;
        float bqx = 0.f, bqy = 0.f, bqz = 0.f;
        if (xlo <= xhi && ylo <= yhi && zlo <= zhi) {
            float shx = 0.f, shy = 0.f, shz = 0.f, thr = FLT_MAX;
            double E1 = 0.0;
            if (PREFILTER) {
                shx = __double2float_rn(sx);
                shy = __double2float_rn(sy);
                shz = __double2float_rn(sz);
                E1 = (fabs(sx - (double)shx) + fabs(sy - (double)shy) + fabs(sz - (double)shz)) *
                     (1.0 + 9.5367431640625e-07);
                thr = prefilter_thr(r2, E1, a.dmax, a.inv_dmax);
            }
            for (int z = zlo; z <= zhi; ++z) {
                for (int y = ylo; y <= yhi; ++y) {
                    // one x-row = up to two contiguous ranges of the sorted target
                    int b0, e0, b1 = 0, e1 = 0;
                    if (!g.hashed) {
                        const int64_t base = grid_index_dense(g, 0, y, z);
                        b0 = __ldg(&a.cell_start[base + xlo]);
                        e0 = __ldg(&a.cell_start[base + xhi + 1]);
                    } else {
                        const uint32_t s0 = (grid_row_hash(y, z) + (uint32_t)xlo) & g.hmask;
                        const uint32_t cnt = (uint32_t)(xhi - xlo + 1);
                        b0 = __ldg(&a.cell_start[s0]);
                        if ((uint64_t)s0 + cnt <= (uint64_t)g.hmask + 1) {
                            e0 = __ldg(&a.cell_start[s0 + cnt]);
                        } else {
                            e0 = __ldg(&a.cell_start[(int64_t)g.hmask + 1]);
                            b1 = __ldg(&a.cell_start[0]);
                            e1 = __ldg(&a.cell_start[(s0 + cnt) & g.hmask]);
                        }
                    }
                    for (int seg = 0; seg < 2; ++seg) {
                        const int jb = seg ? b1 : b0, je = seg ? e1 : e0;
                        for (int j = jb; j < je; ++j) {
                            const float4 t = __ldg(&a.tpos[j]);
                            if (PREFILTER) {
                                const float ux = t.x - shx, uy = t.y - shy, uz = t.z - shz;
                                const float df = fmaf(uz, uz, fmaf(uy, uy, ux * ux));
                                if (df > thr) continue;
                            }
                            // exact rule (R1-R3): fp64, ((dx dx + dy dy) + dz dz), no FMA
                            const double dx = __dsub_rn(sx, (double)t.x);
                            const double dy = __dsub_rn(sy, (double)t.y);
                            const double dz = __dsub_rn(sz, (double)t.z);
                            const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                                        __dmul_rn(dz, dz));
                            const int idx = __float_as_int(t.w);
                            if (d2 <= r2 && (d2 < best_d2 || (d2 == best_d2 && idx < best_idx))) {
                                best_d2 = d2;
                                best_j = j;
                                best_idx = idx;
                                bqx = t.x, bqy = t.y, bqz = t.z;
                                if (PREFILTER) thr = prefilter_thr(best_d2, E1, a.dmax, a.inv_dmax);
                            }
                        }
                    }
                }
            }
        }
        if (WRITE_CORR) a.corr_out[__float_as_int(p.w)] = best_j >= 0 ? best_idx : -1;
        if (best_j >= 0) {
            // A5: r = (s' - q).n, J = [s' x n ; n] (R4). FMA allowed here.
            const float4 nf = __ldg(&a.tnrm[best_j]);
            const double nx = nf.x, ny = nf.y, nz = nf.z;
            const double r = (sx - (double)bqx) * nx + (sy - (double)bqy) * ny + (sz - (double)bqz) * nz;
            const double J[6] = {sy * nz - sz * ny, sz * nx - sx * nz, sx * ny - sy * nx, nx, ny, nz};
            int k = 0;
#pragma unroll
            for (int u = 0; u < 6; ++u)
#pragma unroll
                for (int v = u; v < 6; ++v) acc[k++] += J[u] * J[v];
#pragma unroll
            for (int u = 0; u < 6; ++u) acc[21 + u] += J[u] * r;
            acc[27] += 1.0;
            acc[28] += best_d2;
        }
    }

    // A6: warp butterfly (fixed order) -> per-warp smem -> fixed-order block sum
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kTerms; ++k) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[warp][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < kTermStride) {
        double s = 0.0;
        if (threadIdx.x < kTerms)
            for (int w = 0; w < kK3Threads / 32; ++w) s += red[w][threadIdx.x];
        a.block_partials[(size_t)blockIdx.x * kTermStride + threadIdx.x] = s;
    }
}

template <bool P, bool W>
static int occ_of() {
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k3_corr_reduce<P, W>, kK3Threads, 0);
    return b;
}

int k3_max_blocks_per_sm(bool prefilter, bool write_corr) {
    if (prefilter) return write_corr ? occ_of<true, true>() : occ_of<true, false>();
    return write_corr ? occ_of<false, true>() : occ_of<false, false>();
}

void launch_k3(const K3Args& a, int blocks, bool prefilter, bool write_corr, cudaStream_t s) {
    if (prefilter) {
        if (write_corr) k3_corr_reduce<true, true><<<blocks, kK3Threads, 0, s>>>(a);
        else k3_corr_reduce<true, false><<<blocks, kK3Threads, 0, s>>>(a);
    } else {
        if (write_corr) k3_corr_reduce<false, true><<<blocks, kK3Threads, 0, s>>>(a);
        else k3_corr_reduce<false, false><<<blocks, kK3Threads, 0, s>>>(a);
    }
}

// ------------------------------------------------------------------- K4
// 6x6 LDL^T without pivoting (R6): singular if any D_k <= 1e-12 max_i A_ii.
__device__ static bool ldlt6_solve(const double* A, const double* b, double* x) {
    double L[6][6], D[6];
    double amax = 0.0;
    for (int i = 0; i < 6; ++i) amax = fmax(amax, A[6 * i + i]);
    if (!(amax > 0.0)) return false;
    for (int j = 0; j < 6; ++j) {
        double d = A[6 * j + j];
        for (int k = 0; k < j; ++k) d -= L[j][k] * L[j][k] * D[k];
        if (!(d > 1e-12 * amax)) return false;
        D[j] = d;
        for (int i = j + 1; i < 6; ++i) {
            double v = A[6 * i + j];
            for (int k = 0; k < j; ++k) v -= L[i][k] * L[j][k] * D[k];
            L[i][j] = v / d;
        }
    }
    double y[6];
    for (int i = 0; i < 6; ++i) {
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
        y[i] = v;
    }
    for (int i = 5; i >= 0; --i) {
        double v = y[i] / D[i];
        for (int k = i + 1; k < 6; ++k) v -= L[k][i] * x[k];
        x[i] = v;
    }
    return true;
}

// exp of the twist xi = (w, v) (R5): Rodrigues R and the left Jacobian V.
__device__ static void se3_exp(const double* xi, double* E /*3x4*/) {
    const double wx = xi[0], wy = xi[1], wz = xi[2];
    const double t2 = wx * wx + wy * wy + wz * wz, t = sqrt(t2);
    double A, B, C;
    if (t < 1e-6) {
        A = 1.0 - t2 / 6.0;
        B = 0.5 - t2 / 24.0;
        C = 1.0 / 6.0 - t2 / 120.0;
    } else {
        double s, c;
        sincos(t, &s, &c);
        A = s / t;
        B = (1.0 - c) / t2;
        C = (t - s) / (t2 * t);
    }
    const double W[3][3] = {{0, -wz, wy}, {wz, 0, -wx}, {-wy, wx, 0}};
    for (int i = 0; i < 3; ++i) {
        double Vv = 0.0;
        for (int j = 0; j < 3; ++j) {
            double w2 = W[i][0] * W[0][j] + W[i][1] * W[1][j] + W[i][2] * W[2][j];
            double I = (i == j) ? 1.0 : 0.0;
            E[4 * i + j] = I + A * W[i][j] + B * w2;
            Vv += (I + B * W[i][j] + C * w2) * xi[3 + j];
        }
        E[4 * i + 3] = Vv;
    }
}

__global__ void __launch_bounds__(kTailThreads)
    k_tail(const double* __restrict__ partials, int nblocks, double* gathered, int world, int rank,
           IcpState* st, double* hist_fit, double* hist_rmse, int mode) {
    __shared__ double terms[kTermStride];
    if (!(mode & TAIL_STEP) && st->done) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (mode & TAIL_REDUCE_BLOCKS) {
        if (warp < kTerms) {
            double s = 0.0;
            for (int b = lane; b < nblocks; b += 32) s += partials[(size_t)b * kTermStride + warp];
#pragma unroll
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) terms[warp] = s;
        }
        __syncthreads();
        if (mode & TAIL_WRITE_RANK) {
            if (threadIdx.x < kTermStride)
                gathered[rank * kTermStride + threadIdx.x] = threadIdx.x < kTerms ? terms[threadIdx.x] : 0.0;
            return;
        }
    }
    if (mode & TAIL_SUM_RANKS) {
        if (threadIdx.x < kTerms) {
            double s = 0.0;
            for (int r = 0; r < world; ++r) s += gathered[r * kTermStride + threadIdx.x];
            terms[threadIdx.x] = s;
        }
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    for (int k = 0; k < kTerms; ++k) st->terms[k] = terms[k];
    if (mode & TAIL_STEP) return;

    // A8: criteria (R7, R8) then the Gauss-Newton update (Eq. 2, R5, R6)
    const double cnt = terms[27];
    const double fit = cnt / st->n_total;
    const double rmse = cnt > 0.0 ? sqrt(terms[28] / cnt) : 0.0;
    const int p = st->passes;
    if (p < st->hist_cap) {
        hist_fit[p] = fit;
        hist_rmse[p] = rmse;
    }
    st->passes = p + 1;
    st->fit = fit;
    st->rmse = rmse;
    int done = 0;
    if (p > 0 && fabs(fit - st->fit_prev) < st->rel_fit && fabs(rmse - st->rmse_prev) < st->rel_rmse) {
        st->converged = 1;
        done = 1;
    }
    st->fit_prev = fit;
    st->rmse_prev = rmse;
    if (!done) {
        if (st->it >= st->max_it || cnt == 0.0) {
            done = 1;
        } else {
            double A[36], b[6], xi[6];
            int k = 0;
            for (int u = 0; u < 6; ++u)
                for (int v = u; v < 6; ++v) {
                    A[6 * u + v] = terms[k];
                    A[6 * v + u] = terms[k];
                    ++k;
                }
            for (int u = 0; u < 6; ++u) b[u] = -terms[21 + u];
            if (cnt < 6.0 || !ldlt6_solve(A, b, xi)) {
                st->flags |= 2;  // O3G_FLAG_DEGENERATE
                done = 1;
            } else {
                double E[12], Tn[12];
                se3_exp(xi, E);
                for (int i = 0; i < 3; ++i)
                    for (int j = 0; j < 4; ++j)
                        Tn[4 * i + j] = E[4 * i + 0] * st->T[j] + E[4 * i + 1] * st->T[4 + j] +
                                        E[4 * i + 2] * st->T[8 + j] + (j == 3 ? E[4 * i + 3] : 0.0);
                for (int q = 0; q < 12; ++q) st->T[q] = Tn[q];
                st->T[12] = 0.0, st->T[13] = 0.0, st->T[14] = 0.0, st->T[15] = 1.0;
                st->it += 1;
            }
        }
    }
    if (done && cnt == 0.0) st->flags |= 1;  // O3G_FLAG_NO_CORRESPONDENCES
    st->done = done;
}

void launch_tail(const double* partials, int nblocks, double* gathered, int world, int rank,
                 IcpState* st, double* hist_fit, double* hist_rmse, int mode, cudaStream_t s) {
    k_tail<<<1, kTailThreads, 0, s>>>(partials, nblocks, gathered, world, rank, st, hist_fit,
                                      hist_rmse, mode);
}

}  // namespace o3g
