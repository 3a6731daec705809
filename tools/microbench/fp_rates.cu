// fp_rates.cu — B200 microbenchmark of the arithmetic the correspondence
// kernel leans on (SURVEY §8(d) asks for it; MEASURED_PEAKS has only HBM and
// bf16): dependent-chain-free DADD / DMUL / DFMA / F2F.F64.F32 / FFMA / FFMA2
// throughput per SM, in operations per clock. Not part of the library.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp_rates fp_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;   // independent chains per thread (hides latency)

template <int OP>
__global__ void k_rate(double* out, float* outf, double seed) {
    double d[kChains];
    float f[kChains * 2];
    for (int c = 0; c < kChains; ++c) d[c] = seed + threadIdx.x + c, f[2 * c] = (float)d[c], f[2 * c + 1] = (float)(d[c] * 0.5);
    const double a = 1.0000001, b = 1e-9;
    const float af = 1.0000001f, bf = 1e-9f;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == 0) d[c] = __dadd_rn(d[c], b);
            if (OP == 1) d[c] = __dmul_rn(d[c], a);
            if (OP == 2) d[c] = __fma_rn(d[c], a, b);
            if (OP == 3) d[c] += (double)f[c];          // F2F.F64.F32 + DADD
            if (OP == 4) f[c] = __fmaf_rn(f[c], af, bf);
            if (OP == 5) {
                float2 v = make_float2(f[2 * c], f[2 * c + 1]);
                v = __ffma2_rn(v, make_float2(af, af), make_float2(bf, bf));
                f[2 * c] = v.x, f[2 * c + 1] = v.y;
            }
            if (OP == 3) f[c] = __fadd_rn(f[c], bf);      // keep the conversion input changing
        }
    }
    double s = 0.0;
    float sf = 0.f;
    for (int c = 0; c < kChains; ++c) s += d[c], sf += f[2 * c] + f[2 * c + 1];
    if (s == 123.456) out[0] = s;
    if (sf == 123.456f) outf[0] = sf;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);   // kHz (max)
    double* out;
    float* outf;
    cudaMalloc(&out, 8);
    cudaMalloc(&outf, 4);
    const char* names[] = {"DADD", "DMUL", "DFMA", "F2F.F64.F32(+DADD)", "FFMA", "FFMA2 (2 lanes/op)"};
    const int blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](int op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (op) {
                case 0: k_rate<0><<<blocks, threads>>>(out, outf, 1.0); break;
                case 1: k_rate<1><<<blocks, threads>>>(out, outf, 1.0); break;
                case 2: k_rate<2><<<blocks, threads>>>(out, outf, 1.0); break;
                case 3: k_rate<3><<<blocks, threads>>>(out, outf, 1.0); break;
                case 4: k_rate<4><<<blocks, threads>>>(out, outf, 1.0); break;
                default: k_rate<5><<<blocks, threads>>>(out, outf, 1.0); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * kIters * kChains * (op == 5 ? 2 : 1);
        const double rate = ops / (ms * 1e-3);
        printf("%-22s %8.3f Tops/s  %7.1f ops/clk/SM (at %d MHz max clock)\n", names[op], rate / 1e12,
               rate / sms / (clk * 1e3), clk / 1000);
    };
    for (int op = 0; op < 6; ++op) run(op);
    printf("SMs %d\n", sms);
    return cudaGetLastError() != cudaSuccess;
}
