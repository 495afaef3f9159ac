// trace.cu — selection traces and head-stability overlaps.
//
// fc_trace_capture copies every (row, layer, head)'s current top-K selection
// into a device trace buffer laid out exactly as the FXTK records
// (trace.py:1-19: per step, L*H records of K u32, layer-major, head-minor),
// so a whole profiling run lands in HBM inside the step graph and leaves in
// one D2H copy.
//
// fc_trace_overlap computes |anchor ∩ later| for every (layer, head, window,
// offset) — the integer core of the random-corrected overlap
// (stability.py:24-62): one CTA per (window, layer, head) sets the anchor's
// pages in a shared-memory bitmap, and each warp counts the members of one
// later step's selection with ballots.  The float64 RCO / mean arithmetic
// stays on the host so it is bit-identical to the reference.
#include "launchers.cuh"
#include "store.cuh"

namespace fc {

constexpr int kTraceThreads = 128;

__global__ void __launch_bounds__(kTraceThreads)
trace_capture_kernel(StoreView s, uint32_t *tsel, uint32_t *tpool, int step_base, int n_slots,
                     int topk, int extra_tokens) {
    const int slot = *s.step - step_base;
    if (slot < 0 || slot >= n_slots) return;
    const int lhn = s.L * s.H;
    const int b = blockIdx.x / lhn, lh = blockIdx.x % lhn;
    const int hx = s.hix(b, lh / s.H, lh % s.H);
    const int n = s.n_sel[hx];
    const int32_t *src = s.sel + (int64_t)hx * s.SELCAP;
    uint32_t *dst = tsel + (((int64_t)b * n_slots + slot) * lhn + lh) * topk;
    if (n < topk) {  // a record needs exactly K pages: pool <= K is not traceable
        if (threadIdx.x == 0) set_error(s.err, FC_ERR_TRACE_SHORT);
        for (int i = threadIdx.x; i < topk; i += blockDim.x) dst[i] = 0xffffffffu;
    } else {
        for (int i = threadIdx.x; i < topk; i += blockDim.x) dst[i] = (uint32_t)src[i];
    }
    if (lh == 0 && threadIdx.x == 0) {
        const int n_tok = s.seq_len[b] + extra_tokens;
        tpool[(int64_t)b * n_slots + slot] = (uint32_t)((n_tok + s.PS - 1) / s.PS);
    }
}

// grid (n_windows * L * H); inter [L][H][n_windows][window-1], -1 = degenerate
// pool (N_t <= K) at the later step
__global__ void __launch_bounds__(kTraceThreads)
trace_overlap_kernel(const uint32_t *__restrict__ sel, const uint32_t *__restrict__ pool, int L, int H,
                     int K, const int32_t *__restrict__ starts, int n_windows, int window, int words,
                     int32_t *inter) {
    extern __shared__ uint32_t bitmap[];
    const int lh = blockIdx.x % (L * H), w = blockIdx.x / (L * H);
    const int start = starts[w];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < words; i += blockDim.x) bitmap[i] = 0u;
    __syncthreads();
    const uint32_t *anchor = sel + ((int64_t)start * L * H + lh) * K;
    for (int i = tid; i < K; i += blockDim.x) {
        const uint32_t p = anchor[i];
        if ((p >> 5) < (uint32_t)words) atomicOr(&bitmap[p >> 5], 1u << (p & 31));
    }
    __syncthreads();
    int32_t *row = inter + ((int64_t)lh * n_windows + w) * (window - 1);
    for (int d = 1 + wid; d < window; d += kTraceThreads / 32) {
        const int t = start + d;
        if (pool[t] <= (uint32_t)K) {
            if (lane == 0) row[d - 1] = -1;
            continue;
        }
        const uint32_t *later = sel + ((int64_t)t * L * H + lh) * K;
        int cnt = 0;
        for (int i0 = 0; i0 < K; i0 += 32) {
            const int i = i0 + lane;
            bool hit = false;
            if (i < K) {
                const uint32_t p = later[i];
                hit = (p >> 5) < (uint32_t)words && ((bitmap[p >> 5] >> (p & 31)) & 1u);
            }
            cnt += __popc(__ballot_sync(0xffffffffu, hit));
        }
        if (lane == 0) row[d - 1] = cnt;
    }
}

cudaError_t launch_trace_capture(const StoreView &s, uint32_t *tsel, uint32_t *tpool, int step_base,
                                 int n_slots, int topk, int extra, int batch, cudaStream_t st) {
    if (batch == 0) return cudaSuccess;
    trace_capture_kernel<<<batch * s.L * s.H, kTraceThreads, 0, st>>>(s, tsel, tpool, step_base, n_slots,
                                                                       topk, extra);
    return cudaGetLastError();
}

cudaError_t launch_trace_overlap(const uint32_t *sel, const uint32_t *pool, int L, int H, int K,
                                 const int32_t *starts, int n_windows, int window, int max_pool,
                                 int32_t *inter, cudaStream_t st) {
    const int words = (max_pool + 31) / 32;
    const size_t smem = (size_t)words * sizeof(uint32_t);
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(trace_overlap_kernel,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    trace_overlap_kernel<<<n_windows * L * H, kTraceThreads, smem, st>>>(sel, pool, L, H, K, starts,
                                                                         n_windows, window, words, inter);
    return cudaGetLastError();
}

}  // namespace fc
