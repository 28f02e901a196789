// Microbenchmark: random 8-byte gathers from a price vector held in
// distributed shared memory (each CTA of a cluster holds a slice) vs L2.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int U>
__global__ void dsm(const int *__restrict__ idx, long long n, int slice, double *out) {
    extern __shared__ double ps[];
    cg::cluster_group cl = cg::this_cluster();
    const int csz = cl.num_blocks();
    for (int i = threadIdx.x; i < slice; i += blockDim.x) ps[i] = 1e-9 * i;
    cl.sync();
    double acc = 0.0;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long long k = i + u * stride;
            int j = k < n ? idx[k] : 0;
            int r = j / slice, o = j - r * slice;
            const double *rp = cl.map_shared_rank(ps, r % csz);
            v[u] = rp[o];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    cl.sync();
    if (acc == 1.2345) *out = acc;
}

int main() {
    const long long n = 1LL << 27;
    const int m = 100000;
    int *idx;
    double *out;
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 8);
    int *h = (int *)malloc(n * 4);
    unsigned long long s = 88172645463325252ull;
    for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % m); }
    cudaMemcpy(idx, h, n * 4, cudaMemcpyHostToDevice);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int csz : {8, 16}) {
        for (int w : {8, 16, 32}) {
            auto run = [&](auto kern, const char *nm) {
                const int slice = (m + csz - 1) / csz;
                size_t sm = (size_t)slice * 8;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                if (csz > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                cudaLaunchConfig_t cfg = {};
                int grid = (nsm / csz) * csz;
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(w * 32);
                cfg.dynamicSmemBytes = sm;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = csz; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                cfg.attrs = at; cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, kern, (const int *)idx, n, slice, out);
                cudaEventRecord(e0);
                cudaLaunchKernelEx(&cfg, kern, (const int *)idx, n, slice, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("cluster %2d grid %3d warps/SM %2d %s: %.3f ms  %.3g gathers/s  %.3f /clk/SM (%s)\n", csz, grid, w, nm,
                       ms, n / (ms * 1e-3), n / (ms * 1e-3) / grid / 1.965e9, cudaGetErrorString(cudaGetLastError()));
            };
            run(dsm<4>, "U4");
            run(dsm<8>, "U8");
        }
    }
    return 0;
}
