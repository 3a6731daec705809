// normals.cu — estimate_normals on the device (SPEC
// S:67-75; "estimate_normals(downpcd, KDTreeSearchParamHybrid(
// radius = 0.1, max_nn = 30))" and PAPER.md:238, the paper's own example of
// an `omp for` loop).
//
// The cloud is indexed by the same voxel-hash grid as the ICP target (cell =
// radius), one thread per point in grid order. The hybrid neighbourhood is
// the max_nn nearest points within the radius under the ICP pass's exact
// rule (fp64 d^2 from fp32, ((dx dx + dy dy) + dz dz), no FMA, inclusive,
// ties -> lower original index), kept in a bounded list, then ordered by
// (d^2, index). Mean and covariance are summed in that order in fp64 without
// contraction (bit-identical to a sequential sum), and the normal is the
// unit eigenvector of the smallest eigenvalue (Jacobi), its largest-magnitude
// component made positive. Fewer than 3 neighbours -> (0,0,1), counted.
#include "o3g_internal.cuh"

namespace o3g {

constexpr int kMaxNN = 64;

__device__ static void jacobi_sym3(double* A, double* w, double* V) {
    for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
    for (int sweep = 0; sweep < 64; ++sweep) {
        const double off = fabs(A[1]) + fabs(A[2]) + fabs(A[5]);
        const double dia = fabs(A[0]) + fabs(A[4]) + fabs(A[8]);
        if (off <= 1e-300 || off <= 1e-18 * dia) break;
        for (int p = 0; p < 2; ++p)
            for (int q = p + 1; q < 3; ++q) {
                const double apq = A[3 * p + q];
                if (apq == 0.0) continue;
                const double th = (A[3 * q + q] - A[3 * p + p]) / (2.0 * apq);
                const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
                for (int k = 0; k < 3; ++k) {
                    const double akp = A[3 * k + p], akq = A[3 * k + q];
                    A[3 * k + p] = c * akp - sn * akq;
                    A[3 * k + q] = sn * akp + c * akq;
                }
                for (int k = 0; k < 3; ++k) {
                    const double apk = A[3 * p + k], aqk = A[3 * q + k];
                    A[3 * p + k] = c * apk - sn * aqk;
                    A[3 * q + k] = sn * apk + c * aqk;
                }
                for (int k = 0; k < 3; ++k) {
                    const double vkp = V[3 * k + p], vkq = V[3 * k + q];
                    V[3 * k + p] = c * vkp - sn * vkq;
                    V[3 * k + q] = sn * vkp + c * vkq;
                }
            }
    }
    for (int i = 0; i < 3; ++i) w[i] = A[4 * i];
}

__device__ __forceinline__ bool nb_less(double da, int ia, double db, int ib) {
    return da < db || (da == db && ia < ib);
}

__global__ void k_normals(const float4* __restrict__ tpos, int n, const int32_t* __restrict__ cs,
                          GridDev g, double r2, int max_nn, float* __restrict__ out,
                          int32_t* __restrict__ nbr_count, unsigned long long* fallback) {
    double hd[kMaxNN];
    int hi[kMaxNN], hj[kMaxNN];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 p = __ldg(&tpos[i]);
        const int oidx = __float_as_int(p.w);
        const double sx = p.x, sy = p.y, sz = p.z;
        const int cx = cell_coord(sx, g.ox, g.inv_h, g.nx), cy = cell_coord(sy, g.oy, g.inv_h, g.ny),
                  cz = cell_coord(sz, g.oz, g.inv_h, g.nz);
        const int xlo = max(cx - 1, 0), xhi = min(cx + 1, g.nx - 1);
        int cnt = 0, worst = 0;
        for (int z = max(cz - 1, 0); z <= min(cz + 1, g.nz - 1); ++z)
            for (int y = max(cy - 1, 0); y <= min(cy + 1, g.ny - 1); ++y) {
                int b0, e0, b1 = 0, e1 = 0;
                if (!g.hashed) {
                    const int64_t rb = grid_index_dense(g, 0, y, z);
                    b0 = cs[rb + xlo];
                    e0 = cs[rb + xhi + 1];
                } else {
                    const uint32_t s0 = (grid_row_hash(y, z) + (uint32_t)xlo) & g.hmask;
                    const uint32_t w = (uint32_t)(xhi - xlo + 1);
                    b0 = cs[s0];
                    if ((uint64_t)s0 + w <= (uint64_t)g.hmask + 1) {
                        e0 = cs[s0 + w];
                    } else {
                        e0 = cs[(int64_t)g.hmask + 1];
                        b1 = cs[0];
                        e1 = cs[(s0 + w) & g.hmask];
                    }
                }
                for (int seg = 0; seg < 2; ++seg)
                    for (int j = seg ? b1 : b0; j < (seg ? e1 : e0); ++j) {
                        const float4 t = __ldg(&tpos[j]);
                        const double dx = __dsub_rn(sx, (double)t.x), dy = __dsub_rn(sy, (double)t.y),
                                     dz = __dsub_rn(sz, (double)t.z);
                        const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                                    __dmul_rn(dz, dz));
                        if (!(d2 <= r2)) continue;
                        const int idx = __float_as_int(t.w);
                        bool dup = false;   // a hashed row can visit a cell twice
                        if (g.hashed)
                            for (int u = 0; u < cnt; ++u) dup |= hj[u] == j;
                        if (dup) continue;
                        if (cnt < max_nn) {
                            hd[cnt] = d2, hi[cnt] = idx, hj[cnt] = j;
                            if (cnt == 0 || nb_less(hd[worst], hi[worst], d2, idx)) worst = cnt;
                            ++cnt;
                        } else if (nb_less(d2, idx, hd[worst], hi[worst])) {
                            hd[worst] = d2, hi[worst] = idx, hj[worst] = j;
                            for (int u = 0; u < cnt; ++u)
                                if (nb_less(hd[worst], hi[worst], hd[u], hi[u])) worst = u;
                        }
                    }
            }
        for (int u = 1; u < cnt; ++u) {   // order by (d2, index)
            const double d = hd[u];
            const int ii = hi[u], jj = hj[u];
            int v = u - 1;
            while (v >= 0 && nb_less(d, ii, hd[v], hi[v])) {
                hd[v + 1] = hd[v], hi[v + 1] = hi[v], hj[v + 1] = hj[v];
                --v;
            }
            hd[v + 1] = d, hi[v + 1] = ii, hj[v + 1] = jj;
        }
        if (nbr_count) nbr_count[oidx] = cnt;
        float o0 = 0.f, o1 = 0.f, o2 = 1.f;
        if (cnt < 3) {
            atomicAdd(fallback, 1ull);
        } else {
            double m0 = 0.0, m1 = 0.0, m2 = 0.0;
            for (int u = 0; u < cnt; ++u) {
                const float4 q = __ldg(&tpos[hj[u]]);
                m0 = __dadd_rn(m0, (double)q.x), m1 = __dadd_rn(m1, (double)q.y), m2 = __dadd_rn(m2, (double)q.z);
            }
            const double k = (double)cnt;
            m0 = __ddiv_rn(m0, k), m1 = __ddiv_rn(m1, k), m2 = __ddiv_rn(m2, k);
            double C[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            for (int u = 0; u < cnt; ++u) {
                const float4 q = __ldg(&tpos[hj[u]]);
                const double d[3] = {__dsub_rn((double)q.x, m0), __dsub_rn((double)q.y, m1),
                                     __dsub_rn((double)q.z, m2)};
                for (int aa = 0; aa < 3; ++aa)
                    for (int bb = 0; bb < 3; ++bb) C[3 * aa + bb] = __dadd_rn(C[3 * aa + bb], __dmul_rn(d[aa], d[bb]));
            }
            for (int aa = 0; aa < 9; ++aa) C[aa] = __ddiv_rn(C[aa], k);
            double w[3], V[9];
            jacobi_sym3(C, w, V);
            int sm = 0;
            for (int aa = 1; aa < 3; ++aa)
                if (w[aa] < w[sm]) sm = aa;
            const double v0 = V[sm], v1 = V[3 + sm], v2 = V[6 + sm];
            const double nv = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
            const double a0 = fabs(v0), a1 = fabs(v1), a2 = fabs(v2);
            const double big = (a1 > a0) ? ((a2 > a1) ? v2 : v1) : ((a2 > a0) ? v2 : v0);
            const double sg = big < 0.0 ? -1.0 : 1.0;
            o0 = (float)(sg * v0 / nv), o1 = (float)(sg * v1 / nv), o2 = (float)(sg * v2 / nv);
        }
        out[3 * (int64_t)oidx] = o0, out[3 * (int64_t)oidx + 1] = o1, out[3 * (int64_t)oidx + 2] = o2;
    }
}

void launch_normals(const float4* tpos, int n, const int32_t* cs, const GridDev& g, double r2,
                    int max_nn, float* out, int32_t* nbr_count, unsigned long long* fallback,
                    cudaStream_t s) {
    int b = (n + 127) / 128;
    b = b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b);
    k_normals<<<b, 128, 0, s>>>(tpos, n, cs, g, r2, max_nn, out, nbr_count, fallback);
}

}  // namespace o3g
