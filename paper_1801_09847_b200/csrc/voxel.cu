// voxel.cu — voxel_down_sample on the device (SPEC
// S:58-61, Fig. 1 "voxel_down_sample(pcd, voxel_size = 0.05)").
//
// Each output point is the mean of the input points of one occupied voxel of
// the grid anchored at the cloud's minimum bound, voxel index
// floor((p - min) / voxel) per axis (floor semantics); normals are averaged
// the same way and renormalised; output order is ascending lexicographic
// (ix, iy, iz). Reuses the grid machinery of A1: 64-bit voxel keys, a stable
// radix sort of (key, index), run boundaries by scan, then one thread per
// voxel summing its points in original-index order in fp64 (so the result
// is bit-identical to a sequential sum) and rounding the mean once to fp32.
#include "o3g_internal.cuh"

namespace o3g {

__global__ void k_vox_keys(const float* __restrict__ xyz, int64_t n, double mx, double my, double mz,
                           double voxel, uint64_t dy, uint64_t dz, uint64_t* __restrict__ keys,
                           int32_t* __restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t ix = (uint64_t)floor(__ddiv_rn(__dsub_rn((double)xyz[3 * i + 0], mx), voxel));
        const uint64_t iy = (uint64_t)floor(__ddiv_rn(__dsub_rn((double)xyz[3 * i + 1], my), voxel));
        const uint64_t iz = (uint64_t)floor(__ddiv_rn(__dsub_rn((double)xyz[3 * i + 2], mz), voxel));
        keys[i] = (ix * dy + iy) * dz + iz;
        vals[i] = (int32_t)i;
    }
}

__global__ void k_run_flags(const uint64_t* __restrict__ keys, int64_t n, int32_t* __restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_run_starts(const int32_t* __restrict__ flags, const int32_t* __restrict__ runid,
                             int64_t n, int32_t* __restrict__ starts) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (flags[i]) starts[runid[i] - 1] = (int32_t)i;
        if (i == n - 1) starts[runid[i]] = (int32_t)n;
    }
}

__global__ void k_vox_mean(const float* __restrict__ xyz, const float* __restrict__ nrm,
                           const int32_t* __restrict__ vals, const int32_t* __restrict__ starts,
                           int64_t nruns, float* __restrict__ out_xyz, float* __restrict__ out_nrm) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nruns;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = starts[r], e = starts[r + 1];
        double px = 0.0, py = 0.0, pz = 0.0, qx = 0.0, qy = 0.0, qz = 0.0;
        for (int32_t k = s; k < e; ++k) {   // stable sort: original-index order
            const int64_t v = vals[k];
            px = __dadd_rn(px, (double)xyz[3 * v]);
            py = __dadd_rn(py, (double)xyz[3 * v + 1]);
            pz = __dadd_rn(pz, (double)xyz[3 * v + 2]);
            if (nrm) {
                qx = __dadd_rn(qx, (double)nrm[3 * v]);
                qy = __dadd_rn(qy, (double)nrm[3 * v + 1]);
                qz = __dadd_rn(qz, (double)nrm[3 * v + 2]);
            }
        }
        const double cnt = (double)(e - s);
        out_xyz[3 * r + 0] = __double2float_rn(__ddiv_rn(px, cnt));
        out_xyz[3 * r + 1] = __double2float_rn(__ddiv_rn(py, cnt));
        out_xyz[3 * r + 2] = __double2float_rn(__ddiv_rn(pz, cnt));
        if (nrm && out_nrm) {
            const double nn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(qx, qx), __dmul_rn(qy, qy)),
                                                   __dmul_rn(qz, qz)));
            out_nrm[3 * r + 0] = nn > 0.0 ? __double2float_rn(__ddiv_rn(qx, nn)) : 0.f;
            out_nrm[3 * r + 1] = nn > 0.0 ? __double2float_rn(__ddiv_rn(qy, nn)) : 0.f;
            out_nrm[3 * r + 2] = nn > 0.0 ? __double2float_rn(__ddiv_rn(qz, nn)) : 0.f;
        }
    }
}

static int nblk(int64_t n) {
    int64_t b = (n + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

void launch_vox_keys(const float* xyz, int64_t n, const double mn[3], double voxel, uint64_t dy,
                     uint64_t dz, uint64_t* keys, int32_t* vals, cudaStream_t s) {
    k_vox_keys<<<nblk(n), 256, 0, s>>>(xyz, n, mn[0], mn[1], mn[2], voxel, dy, dz, keys, vals);
}
void launch_run_flags(const uint64_t* keys, int64_t n, int32_t* flags, cudaStream_t s) {
    k_run_flags<<<nblk(n), 256, 0, s>>>(keys, n, flags);
}
void launch_run_starts(const int32_t* flags, const int32_t* runid, int64_t n, int32_t* starts,
                       cudaStream_t s) {
    k_run_starts<<<nblk(n), 256, 0, s>>>(flags, runid, n, starts);
}
void launch_vox_mean(const float* xyz, const float* nrm, const int32_t* vals, const int32_t* starts,
                     int64_t nruns, float* out_xyz, float* out_nrm, cudaStream_t s) {
    k_vox_mean<<<nblk(nruns), 256, 0, s>>>(xyz, nrm, vals, starts, nruns, out_xyz, out_nrm);
}

}  // namespace o3g
