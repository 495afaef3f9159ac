// Cycles per page of Bf16Warp<128>::page (the attention inner step) with the
// page already in shared memory (profiling aid): NW warps per CTA, each
// repeatedly attending its own resident page; no global traffic.
#include <cstdio>
#include "../../paper_2511_00868_b200/csrc/attn_warp.cuh"

using namespace fc;

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) page_loop(const __nv_bfloat16 *q, int reps, float *sink,
                                                        long long *cycles) {
    extern __shared__ __align__(128) char ring[];
    constexpr int PB = AttnGeom<__nv_bfloat16, 128>::kPageBytes;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    char *page = ring + (size_t)w * PB;
    for (int i = lane; i < PB / 4; i += 32) reinterpret_cast<uint32_t *>(page)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
    __syncwarp();
    Bf16Warp<128> st;
    st.init(q, 4, lane);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) st.page(page, 16, 0.1f, lane);
    const long long t1 = clock64();
    st.finalize();
    float acc = st.m[0] + st.l[0];
    for (int i = 0; i < 16; ++i) acc += st.acc[i][0];
    if (acc == 1.2345f) sink[0] = acc;
    if (lane == 0) cycles[blockIdx.x * NW + w] = t1 - t0;
}

template <int NW>
void run(const __nv_bfloat16 *q, float *sink, long long *cyc) {
    constexpr int PB = AttnGeom<__nv_bfloat16, 128>::kPageBytes;
    cudaFuncSetAttribute(page_loop<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, NW * PB);
    const int reps = 2000;
    page_loop<NW><<<1, NW * 32, NW * PB>>>(q, reps, sink, cyc);
    cudaDeviceSynchronize();
    long long h[32];
    cudaMemcpy(h, cyc, NW * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < NW; ++i) mx = h[i] > mx ? h[i] : mx;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_page = (double)mx / reps;
    const double gbs = NW * (double)PB / (per_page / (clk * 1e3)) / 1e9;
    printf("warps %2d: %.0f cycles per page per warp -> %.1f GB/s per SM at %d MHz\n", NW, per_page, gbs, clk / 1000);
}

int main() {
    __nv_bfloat16 *q;
    float *sink;
    long long *cyc;
    cudaMalloc(&q, 16 * 128 * 2);
    cudaMemset(q, 0, 16 * 128 * 2);
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, 64 * sizeof(long long));
    run<1>(q, sink, cyc);
    run<4>(q, sink, cyc);
    run<8>(q, sink, cyc);
    run<16>(q, sink, cyc);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
