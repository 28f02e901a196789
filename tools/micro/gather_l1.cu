// Microbenchmark: random 8-byte gathers from an L2-resident 800 KB array
// (the price vector p at config 4) vs the L1 capacity left by the kernel's
// shared-memory allocation, warps per SM and loads in flight per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U, int MODE>
__global__ void gather(const double *__restrict__ x, const int *__restrict__ idx, long long n, double *out) {
    extern __shared__ double pad[];
    double acc = 0.0;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long k = i + u * stride;
            if (MODE == 0) v[u] = k < n ? __ldg(x + idx[k]) : 0.0;
            else v[u] = k < n ? __ldcg(x + idx[k]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 1.2345) { pad[threadIdx.x] = acc; *out = pad[0]; }
}

int main() {
    const long long n = 1LL << 27;
    const long long win = 100000;  // goods
    int *idx;
    double *x, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 8);
    cudaMalloc(&x, win * 8);
    cudaMemset(x, 0, win * 8);
    int *h = (int *)malloc(n * 4);
    unsigned long long s = 88172645463325252ull;
    for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % win); }
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int smems[] = {8, 64, 100, 132, 164, 196, 220};  // KB of shared memory per SM (1 CTA/SM)
    for (int kb : smems) {
        for (int w : {16, 32}) {
            auto run = [&](auto kern, const char *nm) {
                size_t sm = (size_t)kb * 1024 - 1024;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                kern<<<nsm, w * 32, sm>>>(x, idx, n, out);
                cudaEventRecord(e0);
                kern<<<nsm, w * 32, sm>>>(x, idx, n, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("smem %3d KB warps/SM %2d %s: %.3f ms  %.3g gathers/s  %.3f /clk/SM (%s)\n", kb, w, nm, ms,
                       n / (ms * 1e-3), n / (ms * 1e-3) / nsm / 1.965e9, cudaGetErrorString(cudaGetLastError()));
            };
            run(gather<4, 0>, "ldg U4 ");
            run(gather<8, 0>, "ldg U8 ");
            run(gather<8, 1>, "ldcg U8");
        }
    }
    return 0;
}
