// k3_common.cuh — device helpers shared by the correspondence kernels.
#pragma once
#include <float.h>
#include <math_constants.h>

#include "o3g_internal.cuh"

namespace o3g {

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

constexpr int kVW = 36;   // padded row stride (doubles) of the V/W staging

// D = A B + C, m8n8k4, fp64 (legacy mma.sync path; DMMA in SASS)
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// flat C index (row*8+col) of term t (O3G_NTERMS order)
__device__ __forceinline__ int term_cidx(int t) {
    if (t < 21) {
        int k = t, u = 0;
        while (k >= 6 - u) { k -= 6 - u; ++u; }
        return u * 8 + (u + k);
    }
    if (t < 27) return 6 * 8 + (t - 21);
    return t == 27 ? 7 * 8 + 6 : 7 * 8 + 7;
}

// point-to-point term t -> flat C index (-1 = unused slot, stays 0):
// [0..8] sum s'_a q_b = C[a][b], [9..11] sum s' = C[a][3], [12..14] sum q =
// C[3][b], [27] count = C[3][3], [28] sum d2 = C[3][4]
__device__ __forceinline__ int term_cidx_p2p(int t) {
    if (t < 9) return (t / 3) * 8 + (t % 3);
    if (t < 12) return (t - 9) * 8 + 3;
    if (t < 15) return 3 * 8 + (t - 12);
    if (t == 27) return 3 * 8 + 3;
    if (t == 28) return 3 * 8 + 4;
    return -1;
}

}  // namespace o3g
