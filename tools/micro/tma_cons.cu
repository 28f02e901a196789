// Microbenchmark: tile pipeline with consumer warps releasing stages through an
// "empty" mbarrier (as the fused kernel does), vs producer-only.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t ph) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t n, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(dst)), "l"(src), "r"(n), "r"(sa(bar)) : "memory");
}

template <int NCW, int STAGES>
__global__ void pipe(const double *u, const double *x, const double *xb, const int *col, long long ntiles,
                     int tile, int *ctr, unsigned long long *sink, int mode) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int stage_bytes = tile * 28 + 256;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)STAGES * stage_bytes);
    uint64_t *empty = full + STAGES;
    long long *stile = reinterpret_cast<long long *>(empty + STAGES);
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(NCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp == NCW) {
        if (lane) return;
        for (long long j = 0;; ++j) {
            int s = (int)(j % STAGES);
            if (j >= STAGES) wait(&empty[s], (uint32_t)(((j / STAGES) - 1) & 1));
            long long k = atomicAdd(ctr, 1);
            if (k >= ntiles) {
                stile[s] = -1;
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 0;" ::"r"(sa(&full[s])) : "memory");
                break;
            }
            stile[s] = k;
            unsigned char *b = sm + (size_t)s * stage_bytes;
            long long e0 = k * tile;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(tile * 28) : "memory");
            bulk(b, u + e0, tile * 8, &full[s]);
            bulk(b + tile * 8, x + e0, tile * 8, &full[s]);
            bulk(b + tile * 16, xb + e0, tile * 8, &full[s]);
            bulk(b + tile * 24, col + e0, tile * 4, &full[s]);
        }
        return;
    }
    unsigned long long acc = 0;
    for (long long j = 0;; ++j) {
        int s = (int)(j % STAGES);
        wait(&full[s], (uint32_t)((j / STAGES) & 1));
        long long k = stile[s];
        if (k < 0) break;
        const double *su = reinterpret_cast<const double *>(sm + (size_t)s * stage_bytes);
        if (mode >= 1) {  // touch the tile: every lane reads its share of u
            for (int t = warp * 32 + lane; t < tile; t += NCW * 32) acc += (unsigned long long)su[t];
        }
        if (mode >= 2) {  // write x and xbar back (as the solver does)
            for (int t = warp * 32 + lane; t < tile; t += NCW * 32) {
                const_cast<double *>(x)[k * tile + t] = su[t];
                const_cast<double *>(xb)[k * tile + t] = su[t];
            }
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    if (acc == 12345) *sink = acc;
}

int main() {
    const long long n = 1000LL << 20;
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
    const int tile = 2048;
    long long ntiles = n / tile;
    for (int mode = 0; mode < 3; ++mode) {
        auto run = [&](auto kern, int ncw, const char *name) {
            size_t smem = (size_t)3 * (tile * 28 + 256) + 256;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaMemset(ctr, 0, 4);
            kern<<<nsm, (ncw + 1) * 32, smem>>>(u, x, xb, col, ntiles, tile, ctr, sink, mode);
            cudaMemset(ctr, 0, 4);
            cudaEventRecord(e0);
            kern<<<nsm, (ncw + 1) * 32, smem>>>(u, x, xb, col, ntiles, tile, ctr, sink, mode);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double bytes = n * 28.0 + (mode == 2 ? n * 16.0 : 0.0);
            printf("mode %d %s: %.2f ms  %7.1f GB/s %s\n", mode, name, ms, bytes / (ms * 1e-3) / 1e9,
                   cudaGetErrorString(cudaGetLastError()));
        };
        run(pipe<1, 3>, 1, "1 consumer warp ");
        run(pipe<4, 3>, 4, "4 consumer warps");
        run(pipe<15, 3>, 15, "15 consumer warps");
    }
    return 0;
}
