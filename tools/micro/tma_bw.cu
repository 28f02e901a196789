// Microbenchmark: 1-D TMA bulk-copy (cp.async.bulk) streaming bandwidth per
// chunk size / stage count / CTAs per SM.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_stream(const char *src, long long bytes, int chunk, int stages, unsigned long long *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)stages * chunk);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    long long nchunks = bytes / chunk;
    unsigned long long acc = 0;
    if (threadIdx.x == 0) {
        long long j = 0;
        auto issue = [&](long long c, int s) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(chunk) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(sa(sm + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(sa(&bar[s])) : "memory");
        };
        for (int s = 0; s < stages; ++s) {
            long long c = blockIdx.x + (long long)s * gridDim.x;
            if (c < nchunks) issue(c, s);
        }
        for (j = 0;; ++j) {
            long long c = blockIdx.x + j * gridDim.x;
            if (c >= nchunks) break;
            int s = (int)(j % stages);
            uint32_t ph = (uint32_t)((j / stages) & 1);
            asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(&bar[s])), "r"(ph) : "memory");
            acc += sm[(size_t)s * chunk + 64];
            long long cn = c + (long long)stages * gridDim.x;
            if (cn < nchunks) issue(cn, s);
        }
        if (acc == 12345) *sink = acc;
    }
}

int main() {
    long long bytes = 16LL << 30;
    char *src;
    cudaMalloc(&src, bytes);
    cudaMemset(src, 1, bytes);
    unsigned long long *sink;
    cudaMalloc(&sink, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int chunks[] = {16384, 32768, 65536};
    int stages_l[] = {2, 3, 4, 6, 8, 12};
    int ctas[] = {1, 2, 4};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int ci : chunks) for (int st : stages_l) for (int cp : ctas) {
        size_t smem = (size_t)ci * st + 128;
        if (smem * cp > 227 * 1024) continue;
        cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int grid = nsm * cp;
        tma_stream<<<grid, 32, smem>>>(src, bytes, ci, st, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) tma_stream<<<grid, 32, smem>>>(src, bytes, ci, st, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("chunk %6d stages %2d ctas/sm %d : %7.1f GB/s %s\n", ci, st, cp, 3.0 * bytes / (ms * 1e-3) / 1e9,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
    return 0;
}
