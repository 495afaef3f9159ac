// Per-SM streaming, warp-private rings over CONTIGUOUS 1 MiB per CTA (profiling aid):
// NW warps per CTA, each with its own NST-stage ring of `chunk`-byte bulk
// copies of random page-sized blocks, lane 0 issuing; no compute.
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

__global__ void warp_rings(const char *src, size_t n_blocks, int per_warp, int chunk, int nst,
                           unsigned long long *sink) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t bars[32 * 8];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *my = ring + (size_t)w * nst * chunk;
    uint64_t *mb = bars + w * 8;
    if (lane == 0)
        for (int i = 0; i < nst; ++i) mbar_init(&mb[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    uint32_t x = (blockIdx.x * 1024 + w) * 2654435761u + 12345u;
    size_t cur = ((size_t)blockIdx.x * blockDim.x / 32 + w) * per_warp;
    auto nxt = [&]() { (void)x; return cur++; };
    if (lane == 0)
        for (int i = 0; i < nst && i < per_warp; ++i) {
            expect_tx(&mb[i], chunk);
            bulk(my + (size_t)i * chunk, src + nxt() * chunk, chunk, &mb[i]);
        }
    unsigned long long acc = 0;
    for (int i = 0; i < per_warp; ++i) {
        const int s = i % nst;
        wait(&mb[s], (i / nst) & 1);
        acc += my[(size_t)s * chunk + lane * 4];
        __syncwarp();
        if (lane == 0 && i + nst < per_warp) {
            expect_tx(&mb[s], chunk);
            bulk(my + (size_t)s * chunk, src + nxt() * chunk, chunk, &mb[s]);
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    const size_t total = 8ull << 30;
    char *src;
    unsigned long long *sink;
    cudaMalloc(&src, total);
    cudaMemset(src, 1, total);
    cudaMalloc(&sink, 8);
    cudaFuncSetAttribute(warp_rings, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Cfg { int nw, nst, chunk_kb; };
    const Cfg cfgs[] = {{8, 3, 8}, {16, 3, 4}, {16, 2, 4}, {16, 3, 2}, {8, 4, 4}, {4, 3, 16}, {4, 2, 16}, {1, 3, 64}};
    const int grids[] = {1, 32, 128};
    for (const Cfg &c : cfgs)
        for (int g : grids) {
            const int chunk = c.chunk_kb * 1024;
            const size_t smem = (size_t)c.nw * c.nst * chunk;
            if (smem > 200 * 1024) continue;
            const int per_warp = (int)((1ll << 20) / chunk / c.nw);  // 1 MiB per CTA
            const size_t n_blocks = total / chunk;
            warp_rings<<<g, c.nw * 32, smem>>>(src, n_blocks, per_warp, chunk, c.nst, sink);
            cudaEventRecord(a);
            for (int r = 0; r < 3; ++r) warp_rings<<<g, c.nw * 32, smem>>>(src + (size_t)(r + 1) * (512 << 20), n_blocks, per_warp, chunk, c.nst, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double bytes = 3.0 * g * (double)per_warp * c.nw * chunk;
            const double gbs = bytes / (ms * 1e-3) / 1e9;
            printf("warps %2d x %d stages x %2d KB (%3zu KB in ring), ctas %3d: %8.1f GB/s, %6.1f per SM\n", c.nw,
                   c.nst, c.chunk_kb, smem / 1024, g, gbs, gbs / g);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
