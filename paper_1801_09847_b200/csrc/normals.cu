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
// unit eigenvector of the smallest eigenvalue (closed form, eig3_smallest), its largest-magnitude
// component made positive. Fewer than 3 neighbours -> (0,0,1), counted.
#include "o3g_internal.cuh"

namespace o3g {

constexpr int kMaxNN = 64;

// The row cross product of largest norm of M (each row is orthogonal to M's
// null vector; the largest product is the best-conditioned estimate of it).
__device__ static void best_cross(const double* M, double w[3]) {
    double best = -1.0;
    w[0] = 1.0, w[1] = 0.0, w[2] = 0.0;
    for (int i = 0; i < 3; ++i) {
        const double* x = M + 3 * i;
        const double* y = M + 3 * ((i + 1) % 3);
        const double cx = x[1] * y[2] - x[2] * y[1], cy = x[2] * y[0] - x[0] * y[2],
                     cz = x[0] * y[1] - x[1] * y[0];
        const double n2 = cx * cx + cy * cy + cz * cz;
        if (n2 > best) best = n2, w[0] = cx, w[1] = cy, w[2] = cz;
    }
    const double nn = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    if (nn > 0.0) w[0] /= nn, w[1] /= nn, w[2] /= nn;
    else w[0] = 1.0, w[1] = 0.0, w[2] = 0.0;
}

// Unit eigenvector of the smallest eigenvalue of a symmetric 3x3 C, in closed
// form (no iteration; deliberately a different method from the oracle's
// Jacobi sweeps, so the two are independent checks of each other).
// The eigenvalues of B = (C - q I) / p, q = tr(C)/3, p = sqrt(tr((C-qI)^2)/6),
// are 2 cos(phi + 2 pi k / 3), phi = acos(det(B)/2) / 3 in [0, pi/3]
// (trigonometric solution of the depressed characteristic cubic).
//  - phi >= pi/6: the smallest eigenvalue (k = 1) is at least as far from the
//    middle one as the largest is, and insensitive to the rounding of acos
//    near phi = pi/3 (d lambda/d phi = 0 there, the planar case): its
//    eigenvector is the null vector of C - lambda I (best_cross).
//  - phi < pi/6 (the two smallest are the closer pair, e.g. a collinear
//    neighbourhood, where acos's rounding would swamp their gap): the largest
//    eigenvalue (k = 0, again insensitive) gives its eigenvector u, and the
//    2x2 problem of C restricted to u's orthogonal complement is solved
//    exactly by its rotation angle (atan2): the smaller axis is the answer.
// Both branches are accurate to ~eps lambda_max / gap, the conditioning of
// the problem (checked against numpy eigh on planar, collinear, isotropic and
// near-degenerate covariances: angle x relative gap <= 6e-16).
__device__ static void eig3_smallest(const double* C, double v[3]) {
    const double q = (C[0] + C[4] + C[8]) / 3.0;
    const double a = C[0] - q, b = C[4] - q, c = C[8] - q, d = C[1], e = C[5], f = C[2];
    const double p2 = (a * a + b * b + c * c + 2.0 * (d * d + e * e + f * f)) / 6.0;
    const double p = sqrt(p2);
    if (!(p > 0.0)) {   // isotropic: every direction is an eigenvector
        v[0] = 1.0, v[1] = 0.0, v[2] = 0.0;
        return;
    }
    const double det = a * (b * c - e * e) - d * (d * c - e * f) + f * (d * e - b * f);
    const double r = fmin(fmax(det / (2.0 * p2 * p), -1.0), 1.0);
    const double phi = acos(r) / 3.0;
    double M[9];
    if (phi >= 0.52359877559829887308) {   // pi / 6
        const double lam = q + 2.0 * p * cos(phi + 2.0943951023931954923);   // + 2 pi / 3
        for (int i = 0; i < 9; ++i) M[i] = C[i] - (i % 4 == 0 ? lam : 0.0);
        best_cross(M, v);
        return;
    }
    const double lmax = q + 2.0 * p * cos(phi);
    for (int i = 0; i < 9; ++i) M[i] = C[i] - (i % 4 == 0 ? lmax : 0.0);
    double u[3];
    best_cross(M, u);
    // orthonormal basis (e1, e2) of u's complement
    int k = 0;
    if (fabs(u[1]) < fabs(u[k])) k = 1;
    if (fabs(u[2]) < fabs(u[k])) k = 2;
    double e1[3] = {k == 0 ? 1.0 : 0.0, k == 1 ? 1.0 : 0.0, k == 2 ? 1.0 : 0.0};
    const double ue = u[k];
    for (int i = 0; i < 3; ++i) e1[i] -= ue * u[i];
    const double n1 = sqrt(e1[0] * e1[0] + e1[1] * e1[1] + e1[2] * e1[2]);
    for (int i = 0; i < 3; ++i) e1[i] /= n1;
    const double e2[3] = {u[1] * e1[2] - u[2] * e1[1], u[2] * e1[0] - u[0] * e1[2], u[0] * e1[1] - u[1] * e1[0]};
    double Ce1[3], Ce2[3];
    for (int i = 0; i < 3; ++i) {
        Ce1[i] = C[3 * i] * e1[0] + C[3 * i + 1] * e1[1] + C[3 * i + 2] * e1[2];
        Ce2[i] = C[3 * i] * e2[0] + C[3 * i + 1] * e2[1] + C[3 * i + 2] * e2[2];
    }
    const double A00 = e1[0] * Ce1[0] + e1[1] * Ce1[1] + e1[2] * Ce1[2];
    const double A11 = e2[0] * Ce2[0] + e2[1] * Ce2[1] + e2[2] * Ce2[2];
    const double A01 = e1[0] * Ce2[0] + e1[1] * Ce2[1] + e1[2] * Ce2[2];
    double sn, cs;
    sincos(0.5 * atan2(2.0 * A01, A00 - A11), &sn, &cs);   // (cs, sn): the larger axis
    for (int i = 0; i < 3; ++i) v[i] = -sn * e1[i] + cs * e2[i];
    const double nv = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    for (int i = 0; i < 3; ++i) v[i] /= nv;
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
            double v[3];
            eig3_smallest(C, v);
            const double v0 = v[0], v1 = v[1], v2 = v[2];
            const double nv = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
            // sign rule: the largest-magnitude component positive; ties -> the first
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
