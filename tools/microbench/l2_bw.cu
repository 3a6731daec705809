// l2_bw.cu — B200 microbenchmark: L2 read bandwidth of an L2-resident buffer
// (the roofline denominator for the configs whose working set fits the
// 126 MB L2: tiny, depth, LiDAR, fragment; SURVEY §8(d) asks for it).
// Every SM streams a buffer of `mb` MB repeatedly with 16-byte loads
// (ld.global.cg: bypass L1, served by L2); reported bytes/s after warm-up,
// best of 10 CUDA-event-timed runs. Not part of the library.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_read(const float4* __restrict__ p, size_t n, int reps, float* out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    if (acc == 1234.5f) out[0] = acc;   // (keeps the loads alive)
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (double mb : {8.0, 16.0, 32.0, 48.0, 64.0, 96.0, 1024.0}) {
        const size_t n = (size_t)(mb * 1048576.0 / 16.0);
        float4* p;
        float* out;
        cudaMalloc(&p, n * 16);
        cudaMalloc(&out, 4);
        cudaMemset(p, 0, n * 16);
        const int reps = mb >= 1024.0 ? 2 : 20;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k_read<<<sms * 8, 256>>>(p, n, 1, out);
        float best = 1e30f;
        for (int t = 0; t < 10; ++t) {
            cudaEventRecord(a);
            k_read<<<sms * 8, 256>>>(p, n, reps, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("buffer %7.0f MB  read %8.1f GB/s\n", mb, (double)n * 16 * reps / (best * 1e-3) / 1e9);
        cudaFree(p);
        cudaFree(out);
    }
    return 0;
}
