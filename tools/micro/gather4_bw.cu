// Microbenchmark: TMA tile::gather4 for random 8-byte gathers (p[col]) vs LSU gathers.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// each lane issues gather4s (4 random 16-byte rows) into its slice of smem
template <int INFLIGHT>
__global__ void g4(const __grid_constant__ CUtensorMap tmap, const int *__restrict__ rows, long long nrows,
                   int nw, unsigned long long *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm);
    unsigned char *buf = sm + 128;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        for (int s = 0; s < 2; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[2 * w + s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    // work: groups of 4 rows; warp-batch = 32 lanes * INFLIGHT gather4 = 128*INFLIGHT rows
    const long long per_batch = 128LL * INFLIGHT;
    const long long nbatch = nrows / per_batch;
    unsigned long long acc = 0;
    int ph[2] = {0, 0};
    long long it = 0;
    for (long long bb = blockIdx.x * (long long)nw + w; bb < nbatch; bb += (long long)gridDim.x * nw, ++it) {
        const int s = (int)(it & 1);
        unsigned char *dst = buf + ((size_t)(w * 2 + s) * per_batch) * 32;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[2 * w + s])),
                         "r"((int)(per_batch * 16)) : "memory");
        __syncwarp();
        const int *r = rows + bb * per_batch;
#pragma unroll
        for (int q = 0; q < INFLIGHT; ++q) {
            const int g = q * 32 + lane;  // gather4 index within the batch
            const int r0 = r[4 * g], r1 = r[4 * g + 1], r2 = r[4 * g + 2], r3 = r[4 * g + 3];
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(dst + (size_t)g * 128)),
                "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(sa(&bar[2 * w + s]))
                : "memory");
        }
        // wait for the previous batch of this buffer... simple: wait this batch now
        asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(&bar[2 * w + s])), "r"(ph[s]) : "memory");
        ph[s] ^= 1;
        acc += dst[lane * 16];
    }
    if (acc == 12345) *sink = acc;
}

__global__ void lsu(const double *__restrict__ p, const int *__restrict__ rows, long long n, unsigned long long *sink) {
    double acc = 0;
    long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += 8 * stride) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) { long long k = i + u * stride; v[u] = k < n ? __ldg(p + 2 * rows[k]) : 0.0; }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    if (acc == 1.5) *sink = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const long long m2 = 50000;            // rows of 16 B: p of 100k doubles (800 KB)
    const long long n = 1LL << 27;         // gathered rows
    double *p;
    int *rows;
    unsigned long long *sink;
    cudaMalloc(&p, m2 * 16);
    cudaMalloc(&rows, n * 4);
    cudaMalloc(&sink, 8);
    int *h = (int *)malloc(n * 4);
    unsigned long long s = 88172645463325252ull;
    for (long long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (int)(s % m2); }
    cudaMemcpy(rows, h, n * 4, cudaMemcpyHostToDevice);
    cudaMemset(p, 0, m2 * 16);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &qr);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t dims[2] = {2, (cuuint64_t)m2};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, p, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    lsu<<<nsm * 8, 256>>>(p, rows, n, sink);
    cudaEventRecord(e0);
    lsu<<<nsm * 8, 256>>>(p, rows, n, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("LSU gathers: %.3f ms %.3g rows/s (%s)\n", ms, n / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
    int nws[] = {8, 12, 16};
    for (int nw : nws) {
        auto run = [&](auto kern, int inflight) {
            size_t smem = 128 + (size_t)nw * 2 * 128 * inflight * 32;
            if (smem > 227 * 1024) return;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            kern<<<nsm, nw * 32, smem>>>(tm, rows, n, nw, sink);
            cudaEventRecord(e0);
            kern<<<nsm, nw * 32, smem>>>(tm, rows, n, nw, sink);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("gather4 warps/SM %d inflight/lane %d: %.3f ms %.3g rows/s (%s)\n", nw, inflight, ms,
                   n / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
        };
        run(g4<1>, 1);
        run(g4<2>, 2);
        run(g4<4>, 4);
    }
    return 0;
}
