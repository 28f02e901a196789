// Microbenchmark: random 8-byte gathers from an L2-resident window (as the
// fused column sums do) - gathers/s vs warps per SM and loads in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void gather(const double *__restrict__ x, const int *__restrict__ idx, long long n, double *out) {
    double acc = 0.0;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long k = i + u * stride;
            v[u] = k < n ? __ldcg(x + idx[k]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 1.2345) *out = acc;
}

int main() {
    const long long n = 1LL << 28;  // 2.7e8 gathers
    int *idx;
    double *x, *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    long long windows[] = {1LL << 20, 4LL << 20, 16LL << 20, 256LL << 20};  // doubles
    for (long long win : windows) {
        cudaMalloc(&x, win * 8);
        cudaMemset(x, 0, win * 8);
        // random indices in [0, win)
        int *h = (int *)malloc(n * 4);
        unsigned long long s = 88172645463325252ull;
        for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % win); }
        cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
        free(h);
        int wps[] = {8, 16, 32, 64};
        for (int w : wps) {
            int grid = nsm * (w / 8);
            auto run = [&](auto kern, const char *nm) {
                kern<<<grid, 256>>>(x, idx, n, out);
                cudaEventRecord(e0);
                kern<<<grid, 256>>>(x, idx, n, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("window %5lld MB warps/SM %2d %s: %.2f ms  %.3g gathers/s  (%s)\n", win * 8 >> 20, w, nm, ms,
                       n / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
            };
            run(gather<1>, "U1");
            run(gather<8>, "U8");
        }
        cudaFree(x);
    }
    return 0;
}
