// FP64 pipe probe: issue rate of DFMA, DMUL, DADD chains and mixes on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_mix_probe scripts/fp64_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters, double s) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = s + i * 1e-3 + threadIdx.x * 1e-6;
    const double a = 1.0000001, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) x[i] = fma(x[i], a, b);
            if (MODE == 1) x[i] = x[i] * a;
            if (MODE == 2) x[i] = x[i] + b;
            if (MODE == 3) { x[i] = x[i] * a; }             // with mode-3 second half below
            if (MODE == 4) x[i] = fma(x[i], a, -0.0);       // DMUL as DFMA
            if (MODE == 5) x[i] = fma(x[i], 1.0, b);        // DADD as DFMA
        }
        if (MODE == 3) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = x[i] + b;
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += x[i];
    if (MODE >= 6) {  // three distinct, varying register operands per DFMA
        double y[8], z[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) { y[i] = 1.0 + 1e-9 * (i + threadIdx.x); z[i] = 1e-9 * (i + 1); }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 6) x[i] = fma(y[i], z[(i + 1) & 7], x[i]);
                if (MODE == 7) { x[i] = fma(y[i], z[(i + 3) & 7], x[i]); y[i] = fma(z[i], x[(i + 5) & 7], y[i]); z[i] = fma(x[(i + 2) & 7], y[(i + 6) & 7], z[i]); }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) r += x[i] + y[i] + z[i];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <int MODE>
void run(const char* name, int per_iter) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, iters = 20000;
    double* out; cudaMalloc(&out, sizeof(double) * blocks * 256);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<blocks, 256>>>(out, iters, 1.0);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0); k<MODE><<<blocks, 256>>>(out, iters, 1.0); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const double insts = (double)blocks * 256 * iters * per_iter;
    printf("%-28s %.3f ms  %.2f T thread-instr/s  (%.1f lanes/clk/SM at 1.965 GHz)\n", name, best, insts / best / 1e9,
           insts / (best * 1e-3) / sms / 1.965e9);
    cudaFree(out);
}
int main() {
    run<0>("DFMA", 8); run<1>("DMUL", 8); run<2>("DADD", 8); run<3>("DMUL+DFMA+DADD", 24);
    run<4>("DFMA (x*a - 0)", 8); run<5>("DFMA (x*1 + b)", 8);
    run<6>("DFMA 3 regs (y,z fixed)", 8); run<7>("DFMA 3 regs, all varying", 24);
    return 0;
}
