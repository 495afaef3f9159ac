// Per-SM streaming bandwidth with cp.async.bulk into an N-stage ring
// (profiling aid): G CTAs each stream `per_cta` bytes of distinct HBM through
// `stages` x `chunk` bytes of shared memory; warps only acknowledge chunks.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mbar_init(uint64_t *b, int n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(bytes));
}
__device__ __forceinline__ void bulk(void *dst, const void *src, uint32_t bytes, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(b))
                 : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, int phase) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(b)),
        "r"(phase)
        : "memory");
}

__global__ void stream(const char *src, size_t per_cta, int chunk, int stages, unsigned long long *sink, int ways) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t full[16];
    const char *base = src + (size_t)blockIdx.x * per_cta;
    const int n = (int)(per_cta / chunk);
    auto off = [&](int c) { return (size_t)c * chunk; };
    const int issuer = 32 * (ways == 1 ? 0 : 1);  // placeholder
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    for (int c = 0; c < stages && c < n; ++c) {
        if (threadIdx.x == 32 * (c % ways)) {
            expect_tx(&full[c], chunk);
            bulk(ring + (size_t)c * chunk, base + off(c), chunk, &full[c]);
        }
    }
    unsigned long long acc = 0;
    for (int c = 0; c < n; ++c) {
        const int s = c % stages;
        wait(&full[s], (c / stages) & 1);
        acc += ring[(size_t)s * chunk + threadIdx.x * 4];
        __syncthreads();
        if (threadIdx.x == 32 * (s % ways) && c + stages < n) {
            expect_tx(&full[s], chunk);
            bulk(ring + (size_t)s * chunk, base + off(c + stages), chunk, &full[s]);
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    const size_t total = 6ull << 30;
    char *src;
    unsigned long long *sink;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grids[] = {1, 32, 128};
    const int rings_kb[] = {192};
    const int chunks_kb[] = {16, 32, 64};
    for (int g : grids)
        for (int rk : rings_kb)
            for (int ck : chunks_kb) {
                const int chunk = ck * 1024, stages = rk / ck;
                if (stages > 16) continue;
                const size_t per_cta = (size_t)1 << 20;
              for (int ways : {1, 2, 4, 16}) {
                stream<<<g, 512, (size_t)stages * chunk>>>(src, per_cta, chunk, stages, sink, ways);
                cudaEventRecord(a);
                for (int r = 0; r < 5; ++r) stream<<<g, 512, (size_t)stages * chunk>>>(src + (size_t)(r + 1) * (256 << 20), per_cta, chunk, stages, sink, ways);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = 5.0 * g * per_cta / (ms * 1e-3) / 1e9;
                printf("ctas %3d ring %3d KB chunk %2d KB ways %d: %8.1f GB/s total, %6.1f GB/s per SM\n", g, rk, ck, ways, gbs, gbs / g);
              }
            }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
