// Micro-benchmark of the block-wide selection (profiling aid, not product code).
#include "../paper_2511_00868_b200/csrc/score_select.cu"
#include <cstdio>
#include <vector>
#include <random>

using namespace fc;

__global__ void bench_kernel(const float *scores, int n, int kprime, int32_t *out, long long *t) {
    extern __shared__ uint32_t keys[];
    long long t0 = clock64();
    for (int i = threadIdx.x; i < n; i += blockDim.x) keys[i] = score_key(scores[i]);
    __syncthreads();
    long long t1 = clock64();
    block_select<kScoreThreads>(keys, n, kprime, out);
    long long t2 = clock64();
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; }
}

int main() {
    const int n = 2047, kprime = 127;
    std::vector<float> h(n);
    std::mt19937 rng(1);
    std::normal_distribution<float> nd(200.f, 50.f);
    for (auto &x : h) x = nd(rng);
    float *d; int32_t *o; long long *t;
    cudaMalloc(&d, n * 4); cudaMalloc(&o, 4096); cudaMalloc(&t, 16);
    cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
    for (int rep = 0; rep < 3; ++rep) {
        bench_kernel<<<1, kScoreThreads, n * 4>>>(d, n, kprime, o, t);
        long long ht[2];
        cudaMemcpy(ht, t, 16, cudaMemcpyDeviceToHost);
        printf("load %lld cycles, select %lld cycles (%s)\n", ht[0], ht[1], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
