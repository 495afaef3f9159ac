// Microbenchmark of the in-CTA top-K select (block_select, score_select.cu)
// on score rows dumped from the engine (profiling aid): cycles per select for
// 256 and 512 threads, on the real keys and on synthetic keys.
#include "../../paper_2511_00868_b200/csrc/score_select.cu"
#include <cstdio>
#include <vector>
namespace fc { int max_cluster() { return 16; } }

template <int NT>
__global__ void sel_compact_kernel(const float *scores, int n, int kprime, long long *cyc, int32_t *out) {
    __shared__ uint32_t keys[4096];
    __shared__ uint32_t bits[2 * 4096 / 32 + 2];
    for (int i = threadIdx.x; i < n; i += NT) keys[i] = fc::score_key(scores[(int64_t)blockIdx.x * n + i]);
    __syncthreads();
    const long long t0 = clock64();
    fc::block_select_compact<NT>(keys, n, kprime, out + (int64_t)blockIdx.x * kprime, bits);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int NT>
__global__ void sel_kernel(const float *scores, int n, int kprime, long long *cyc, int32_t *out) {
    __shared__ uint32_t keys[4096];
    for (int i = threadIdx.x; i < n; i += NT) keys[i] = fc::score_key(scores[(int64_t)blockIdx.x * n + i]);
    __syncthreads();
    const long long t0 = clock64();
    fc::block_select<NT>(keys, n, kprime, out + (int64_t)blockIdx.x * kprime);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char **argv) {
    FILE *f = fopen(argv[1], "rb");
    int rows = atoi(argv[2]), n = atoi(argv[3]);
    std::vector<float> h((size_t)rows * n);
    fseek(f, atol(argv[4]), SEEK_SET);  // (npy header length)
    size_t got = fread(h.data(), 4, h.size(), f);
    fclose(f);
    if (got != h.size()) { printf("short read %zu\n", got); return 1; }
    float *d; long long *cyc; int32_t *out;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&cyc, rows * 8); cudaMalloc(&out, rows * 128 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    std::vector<long long> c(rows);
    for (int rep = 0; rep < 3; ++rep) {
        sel_kernel<256><<<rows, 256>>>(d, n, 127, cyc, out);
        cudaMemcpy(c.data(), cyc, rows * 8, cudaMemcpyDeviceToHost);
        printf("NT=256:"); for (auto x : c) printf(" %lld", x); printf("\n");
        sel_kernel<512><<<rows, 512>>>(d, n, 127, cyc, out);
        cudaMemcpy(c.data(), cyc, rows * 8, cudaMemcpyDeviceToHost);
        printf("NT=512:"); for (auto x : c) printf(" %lld", x); printf("\n");
        std::vector<int32_t> o1((size_t)rows * 127), o2(o1.size());
        cudaMemcpy(o1.data(), out, o1.size() * 4, cudaMemcpyDeviceToHost);
        sel_compact_kernel<256><<<rows, 256>>>(d, n, 127, cyc, out);
        cudaMemcpy(c.data(), cyc, rows * 8, cudaMemcpyDeviceToHost);
        printf("compact256:"); for (auto x : c) printf(" %lld", x); printf("\n");
        sel_compact_kernel<512><<<rows, 512>>>(d, n, 127, cyc, out);
        cudaMemcpy(c.data(), cyc, rows * 8, cudaMemcpyDeviceToHost);
        printf("compact512:"); for (auto x : c) printf(" %lld", x); printf("\n");
        cudaMemcpy(o2.data(), out, o2.size() * 4, cudaMemcpyDeviceToHost);
        printf("same selection: %d\n", (int)(o1 == o2));
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
