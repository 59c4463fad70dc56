// What the config-1 interpolation's traffic mix (8 B read, 8 B + 4 B written per
// query, nothing else) can reach on this GPU: a kernel that does only that.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/stream_mix_probe scripts/stream_mix_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024) mix(const double2* __restrict__ q, double2* __restrict__ out, int2* __restrict__ idx,
                                            long long npair) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldcs(q + t);
        __stcs(out + t, make_double2(v.x * 2.0, v.y + 1.0));
        __stcs(idx + t, make_int2((int)v.x, (int)v.y));
    }
}
__global__ void __launch_bounds__(1024) copy(const double2* __restrict__ q, double2* __restrict__ out, long long npair) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < npair; t += (long long)gridDim.x * blockDim.x)
        __stcs(out + t, __ldcs(q + t));
}
int main() {
    const long long n = 1ll << 26, npair = n / 2;
    double2 *q, *out; int2* idx; char* flush;
    cudaMalloc(&q, n * 8); cudaMalloc(&out, n * 8); cudaMalloc(&idx, n * 4); cudaMalloc(&flush, 256 << 20);
    cudaMemset(q, 0, n * 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm)
        for (int which = 0; which < 2; ++which) {
            float best = 1e30f;
            for (int r = 0; r < 8; ++r) {
                cudaMemset(flush, r, 256 << 20);
                cudaEventRecord(e0);
                if (which == 0) mix<<<sms * blocks_per_sm, 1024>>>(q, out, idx, npair);
                else copy<<<sms * blocks_per_sm, 1024>>>(q, out, npair);
                cudaEventRecord(e1); cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
            }
            const double bytes = which == 0 ? n * 20.0 : n * 16.0;
            printf("%s, %d CTA/SM x 1024: %.4f ms, %.0f GB/s\n", which == 0 ? "8 B in, 12 B out" : "copy 8 B in, 8 B out",
                   blocks_per_sm, best, bytes / best / 1e6);
        }
    return 0;
}
