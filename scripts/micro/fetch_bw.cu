// Host -> HBM page-gather bandwidth over UVA (profiling aid for fetch_kernel):
// 8 KiB pages gathered from a pinned host buffer into a device pool, by
// (a) per-thread 16-byte loads with U loads in flight, grid capped at G CTAs,
// (b) cp.async.bulk global(host-mapped) -> shared -> global, one page per
// CTA iteration; vs cudaMemcpyAsync of the same bytes contiguous.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int PB = 8192;

template <int U>
__global__ void gather_ld(const char *host, char *pool, const int *src_pages, int n) {
    for (int c = blockIdx.x; c < n; c += gridDim.x) {
        const uint4 *src = reinterpret_cast<const uint4 *>(host + (int64_t)src_pages[c] * PB);
        uint4 *dst = reinterpret_cast<uint4 *>(pool + (int64_t)c * PB);
        for (int i0 = threadIdx.x; i0 < PB / 16; i0 += blockDim.x * U) {
            uint4 r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) { const int i = i0 + u * blockDim.x; if (i < PB / 16) r[u] = src[i]; }
#pragma unroll
            for (int u = 0; u < U; ++u) { const int i = i0 + u * blockDim.x; if (i < PB / 16) dst[i] = r[u]; }
        }
    }
}

// several pages per CTA in flight through shared memory with bulk copies
template <int NP>
__global__ void gather_bulk(const char *host, char *pool, const int *src_pages, int n) {
    extern __shared__ __align__(128) char smem[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;
    for (int c0 = blockIdx.x * NP; c0 < n; c0 += gridDim.x * NP) {
        const int np = min(NP, n - c0);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar_a), "r"(np * PB) : "memory");
            for (int k = 0; k < np; ++k) {
                const char *src = host + (int64_t)src_pages[c0 + k] * PB;
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem + k * PB);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(dst), "l"(src), "r"(PB), "r"(bar_a) : "memory");
            }
        }
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}"
                     :: "r"(bar_a), "r"(phase) : "memory");
        phase ^= 1;
        if (threadIdx.x == 0) {
            for (int k = 0; k < np; ++k) {
                const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem + k * PB);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             :: "l"(pool + (int64_t)(c0 + k) * PB), "r"(s), "r"(PB) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncthreads();
    }
}

int main() {
    const int64_t host_pages = 1 << 17;  // 1 GiB
    const int n = 8192;                  // 64 MiB gathered
    char *host, *pool;
    int *d_idx;
    CK(cudaHostAlloc(&host, host_pages * PB, cudaHostAllocMapped));
    for (int64_t i = 0; i < host_pages * PB; i += 4096) host[i] = (char)i;
    CK(cudaMalloc(&pool, (int64_t)n * PB));
    std::vector<int> idx(n);
    std::mt19937 rng(1);
    for (int i = 0; i < n; ++i) idx[i] = rng() % host_pages;
    CK(cudaMalloc(&d_idx, n * sizeof(int)));
    CK(cudaMemcpy(d_idx, idx.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    char *hdev;
    CK(cudaHostGetDevicePointer(&hdev, host, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto timeit = [&](auto fn, const char *name) {
        fn(); cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); best = ms < best ? ms : best;
        }
        printf("%-32s %7.1f GB/s\n", name, (double)n * PB / (best / 1e3) / 1e9);
    };
    timeit([&] { cudaMemcpyAsync(pool, host, (int64_t)n * PB, cudaMemcpyHostToDevice); }, "memcpy contiguous");
    for (int g : {16, 32, 64, 148, 296, 1184}) {
        char nm[64];
        snprintf(nm, 64, "ld U=4 grid=%d", g);
        timeit([&] { gather_ld<4><<<g, 128>>>(hdev, pool, d_idx, n); }, nm);
        snprintf(nm, 64, "ld U=4 256thr grid=%d", g);
        timeit([&] { gather_ld<4><<<g, 256>>>(hdev, pool, d_idx, n); }, nm);
    }
    cudaFuncSetAttribute(gather_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * PB);
    cudaFuncSetAttribute(gather_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * PB);
    for (int g : {8, 16, 32, 64, 148}) {
        char nm[64];
        snprintf(nm, 64, "bulk NP=4 grid=%d", g);
        timeit([&] { gather_bulk<4><<<g, 32, 4 * PB>>>(hdev, pool, d_idx, n); }, nm);
        snprintf(nm, 64, "bulk NP=8 grid=%d", g);
        timeit([&] { gather_bulk<8><<<g, 32, 8 * PB>>>(hdev, pool, d_idx, n); }, nm);
    }
    CK(cudaGetLastError());
    return 0;
}
