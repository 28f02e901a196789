// Microbenchmark: the fused kernel's tile load pattern (3 f64 arrays + 1 i32
// array per tile, 2048 entries) vs one contiguous stream of the same bytes.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *bar, int hint, uint64_t pol) {
    if (hint)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(sa(dst)), "l"(src), "r"(n), "r"(sa(bar)), "l"(pol) : "memory");
    else
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(dst)), "l"(src), "r"(n), "r"(sa(bar)) : "memory");
}

__global__ void tiles4(const double *u, const double *x, const double *xb, const int *col, long long ntiles,
                       int tile, int stages, int hint, int dyn, int *ctr, unsigned long long *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int stage_bytes = tile * 28 + 256;
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)stages * stage_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    unsigned long long acc = 0;
    long long held[16];
    auto claim = [&](long long j) -> long long { return dyn ? (long long)atomicAdd(ctr, 1) : blockIdx.x + j * gridDim.x; };
    auto issue = [&](long long k, int s) {
        unsigned char *b = sm + (size_t)s * stage_bytes;
        long long e0 = k * tile;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(tile * 28) : "memory");
        bulk(b, u + e0, tile * 8, &bar[s], hint, pol);
        bulk(b + tile * 8, x + e0, tile * 8, &bar[s], 0, pol);
        bulk(b + tile * 16, xb + e0, tile * 8, &bar[s], hint, pol);
        bulk(b + tile * 24, col + e0, tile * 4, &bar[s], hint, pol);
    };
    for (int s = 0; s < stages; ++s) {
        long long k = claim(s);
        held[s] = k;
        if (k < ntiles) issue(k, s);
    }
    for (long long j = 0;; ++j) {
        int s = (int)(j % stages);
        long long k = held[s];
        if (k >= ntiles) break;
        uint32_t ph = (uint32_t)((j / stages) & 1);
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(&bar[s])), "r"(ph) : "memory");
        acc += sm[(size_t)s * stage_bytes + 64];
        long long kn = claim(j + stages);
        held[s] = kn;
        if (kn < ntiles) issue(kn, s);
    }
    if (acc == 12345) *sink = acc;
}

int main() {
    const long long n = 1000LL << 20;  // 1.05e9 entries
    double *u, *x, *xb;
    int *col, *ctr;
    cudaMalloc(&u, n * 8); cudaMalloc(&x, n * 8); cudaMalloc(&xb, n * 8); cudaMalloc(&col, n * 4);
    cudaMalloc(&ctr, 4);
    cudaMemset(u, 1, n * 8); cudaMemset(x, 1, n * 8); cudaMemset(xb, 1, n * 8); cudaMemset(col, 1, n * 4);
    unsigned long long *sink;
    cudaMalloc(&sink, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int tiles[] = {1024, 2048};
    for (int tile : tiles) for (int stages = 2; stages <= 6; ++stages) for (int hint = 0; hint < 2; ++hint)
    for (int dyn = 0; dyn < 2; ++dyn) {
        size_t smem = (size_t)stages * (tile * 28 + 256) + 256;
        if (smem > 227 * 1024) continue;
        cudaFuncSetAttribute(tiles4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        long long ntiles = n / tile;
        cudaMemset(ctr, 0, 4);
        tiles4<<<nsm, 32, smem>>>(u, x, xb, col, ntiles, tile, stages, hint, dyn, ctr, sink);
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(e0);
        tiles4<<<nsm, 32, smem>>>(u, x, xb, col, ntiles, tile, stages, hint, dyn, ctr, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("tile %5d stages %d hint %d dyn %d : %7.1f GB/s (%.2f ms) %s\n", tile, stages, hint, dyn,
               n * 28.0 / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
