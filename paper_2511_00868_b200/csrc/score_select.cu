// score_select.cu — subsystem (2): query-aware page scoring from the min/max
// summaries and exact top-K page selection.
//
// Reference semantics:
//   score_pages  scoring.py:102-111   s_p = sum_i max(q_i*min_i, q_i*max_i)
//   select_topk  scoring.py:164-193   pinned ∪ best others, score desc then
//                                     index asc, budget min(k, n), ascending out
//   rerank_due   scoring.py:196-202   unstable every step, stable at t % R == 0
//
// GQA group score (builder decision): S_{h,p} = sum_g s_p(q_g).
// By the sign-split identity max(q*mn, q*mx) = q⁺*mx + q⁻*mn (mx >= mn) the
// group score is ONE dot product of the page record [min | max] (2d elements)
// with w = [sum_g q_g⁻ | sum_g q_g⁺]: scoring costs one pass over the
// summaries regardless of G and is HBM-bound (2d*e bytes per page).
//
// Selection is a block-wide 4-pass 8-bit radix select on an orderable 32-bit
// key of the fp32 score (-0.0 == +0.0), ties resolved by lowest page index,
// fused into the last CTA to finish scoring a head (threadfence reduction).
#include "store.cuh"
#include <cub/block/block_scan.cuh>

namespace fc {

constexpr int kScoreThreads = 256;
constexpr int kRoundsPerIter = 8;   // pages per lane-slot per iteration (MLP)

// ---------------------------------------------------------------------------
// block-wide exact top-K over keys[0..n) in shared memory.
// Selects the kprime largest (key desc, index asc) and writes their indices in
// ascending order to out[0..kprime).  Requires kprime < n.

template <int NT>
__device__ void block_select(const uint32_t *keys, int n, int kprime, int32_t *out) {
    using Scan = cub::BlockScan<int, NT>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int hist[256];
    __shared__ uint32_t s_prefix;
    __shared__ int s_remaining;
    const int tid = threadIdx.x;
    uint32_t prefix = 0, mask = 0;
    int remaining = kprime;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            const uint32_t k = keys[i];
            if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1);
        }
        __syncthreads();
        // suffix count from the high digit down: cnt_ge(d) = sum_{d' >= d} hist[d']
        // thread t handles digit 255 - t (NT >= 256)
        const int digit = 255 - tid;
        const int c = (tid < 256) ? hist[digit] : 0;
        int incl, total;
        Scan(scan_tmp).InclusiveSum(c, incl, total);
        if (tid < 256) {
            const int above = incl - c;  // keys with a larger digit
            if (above < remaining && incl >= remaining) {
                s_prefix = prefix | ((uint32_t)digit << shift);
                s_remaining = remaining - above;
            }
        }
        __syncthreads();
        prefix = s_prefix;
        remaining = s_remaining;
        mask |= 255u << shift;
        __syncthreads();
    }
    // prefix is the kprime-th largest key; take every larger key and the
    // `remaining` lowest-index keys equal to it.
    const uint32_t T = prefix;
    const int per = (n + NT - 1) / NT;
    const int lo = min(n, tid * per), hi = min(n, lo + per);
    int eq_local = 0, gt_local = 0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t k = keys[i];
        eq_local += (k == T);
        gt_local += (k > T);
    }
    int eq_before, dummy;
    Scan(scan_tmp).ExclusiveSum(eq_local, eq_before, dummy);
    __syncthreads();
    const int take_eq = max(0, min(eq_local, remaining - eq_before));
    int pos, total_sel;
    Scan(scan_tmp).ExclusiveSum(gt_local + take_eq, pos, total_sel);
    int eq_seen = 0;
    for (int i = lo; i < hi; ++i) {
        const uint32_t k = keys[i];
        bool take = k > T;
        if (k == T) {
            take = eq_seen < take_eq;
            ++eq_seen;
        }
        if (take) out[pos++] = i;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// scoring of one chunk of pages by one CTA

template <typename T, int D>
struct ScoreGeom {
    static constexpr int kRecBytes = 2 * D * (int)sizeof(T);     // [min | max]
    static constexpr int kChunks = kRecBytes / 16;                // 16-byte chunks per page
    static constexpr int kLanesPerPage = kChunks < 32 ? kChunks : 32;
    static constexpr int kChunksPerLane = kChunks / kLanesPerPage;
    static constexpr int kPagesPerSlot = 32 / kLanesPerPage;      // pages side by side in a warp
    static constexpr int kPagesPerIter = kPagesPerSlot * kRoundsPerIter;
    static constexpr int kElemsPerChunk = 16 / (int)sizeof(T);
};

template <typename T>
FC_DEVINL void chunk_to_f(const uint4 &c, float *f);
template <>
FC_DEVINL void chunk_to_f<__nv_bfloat16>(const uint4 &c, float *f) {
    f[0] = bf16lo(c.x); f[1] = bf16hi(c.x); f[2] = bf16lo(c.y); f[3] = bf16hi(c.y);
    f[4] = bf16lo(c.z); f[5] = bf16hi(c.z); f[6] = bf16lo(c.w); f[7] = bf16hi(c.w);
}
template <>
FC_DEVINL void chunk_to_f<float>(const uint4 &c, float *f) {
    f[0] = __uint_as_float(c.x); f[1] = __uint_as_float(c.y);
    f[2] = __uint_as_float(c.z); f[3] = __uint_as_float(c.w);
}

// Scores pages [p0, p1) of head hx; w = [sum q⁻ | sum q⁺] in shared memory.
template <typename T, int D>
__device__ void score_range(const StoreView &s, int hx, int p0, int p1, const float *w,
                            float *scores_row) {
    using Gm = ScoreGeom<T, D>;
    constexpr int LPP = Gm::kLanesPerPage, CPL = Gm::kChunksPerLane, EPC = Gm::kElemsPerChunk;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int sub = lane / LPP;       // which page of a slot
    const int cl = lane % LPP;        // chunk lane within a page
    // per-lane coefficients for its chunk(s)
    float coef[CPL][EPC];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < EPC; ++e) coef[c][e] = w[(cl + c * LPP) * EPC + e];
    const char *base = reinterpret_cast<const char *>(s.summ) +
                       (int64_t)hx * s.NCAP * Gm::kRecBytes;
    for (int it0 = p0 + warp * Gm::kPagesPerIter; it0 < p1; it0 += nwarps * Gm::kPagesPerIter) {
        uint4 raw[kRoundsPerIter][CPL];
#pragma unroll
        for (int r = 0; r < kRoundsPerIter; ++r) {
            const int p = it0 + r * Gm::kPagesPerSlot + sub;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                if (p < p1)
                    raw[r][c] = __ldg(reinterpret_cast<const uint4 *>(
                        base + (int64_t)p * Gm::kRecBytes + (cl + c * LPP) * 16));
                else
                    raw[r][c] = make_uint4(0, 0, 0, 0);
            }
        }
        float v[kRoundsPerIter];
#pragma unroll
        for (int r = 0; r < kRoundsPerIter; ++r) {
            float acc = 0.f;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                float f[EPC];
                chunk_to_f<T>(raw[r][c], f);
#pragma unroll
                for (int e = 0; e < EPC; ++e) acc = fmaf(f[e], coef[c][e], acc);
            }
            v[r] = acc;
        }
        // transpose-reduce 8 values over LPP lanes: 3 halving steps then plain
        // butterflies; afterwards lane bits select which round it holds.
        int ridx = 0;
#pragma unroll
        for (int step = 0, dist = LPP / 2, cnt = kRoundsPerIter / 2; step < 3;
             ++step, dist >>= 1, cnt >>= 1) {
            const bool upper = (lane & dist) != 0;
#pragma unroll
            for (int i = 0; i < cnt; ++i) {
                const float send = upper ? v[i] : v[i + cnt];
                const float keep = upper ? v[i + cnt] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, dist);
            }
            if (upper) ridx += cnt;
        }
#pragma unroll
        for (int dist = LPP / 16; dist > 0; dist >>= 1)
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], dist);
        if ((cl & (LPP / 8 - 1)) == 0) {
            const int p = it0 + ridx * Gm::kPagesPerSlot + sub;
            if (p < p1) scores_row[p] = v[0];
        }
    }
}

template <typename T>
__device__ void load_group_coeffs(const StoreView &s, const T *q, int b, int h, float *w) {
    // w[0..D) = sum_g min(q_g, 0) (multiplies the min row); w[D..2D) = sum_g max(q_g, 0)
    for (int i = threadIdx.x; i < s.D; i += blockDim.x) {
        float neg = 0.f, pos = 0.f;
        for (int g = 0; g < s.G; ++g) {
            const float x = Elem<T>::to_f(q[((int64_t)b * s.H * s.G + h * s.G + g) * s.D + i]);
            neg += fminf(x, 0.f);
            pos += fmaxf(x, 0.f);
        }
        w[i] = neg;
        w[s.D + i] = pos;
    }
}

// grid (chunks, batch*H), block kScoreThreads.  do_select = 0: score pages
// [0, n_pages) of every head; do_select = 1: score [0, n_pages-1) of due heads
// and select (last page pinned).
template <typename T, int D>
__global__ void __launch_bounds__(kScoreThreads)
score_select_kernel(StoreView s, int layer, const T *__restrict__ q,
                    const uint8_t *__restrict__ unstable, int period, int force_due,
                    int topk, int extra_tokens, float *scores, int32_t *counters,
                    int do_select, int chunk_pages) {
    extern __shared__ uint32_t dyn_keys[];
    __shared__ float w[2 * D];
    __shared__ int s_last;
    const int bh = blockIdx.y;
    const int b = bh / s.H, h = bh % s.H;
    if (do_select) {
        const bool due = force_due || unstable[layer * s.H + h] || (*s.step % period == 0);
        if (!due) return;
    }
    const int n_tok = s.seq_len[b] + extra_tokens;
    if (n_tok <= 0) return;
    const int n_pages = (n_tok + s.PS - 1) / s.PS;
    const int hx = s.hix(b, layer, h);
    if (do_select && n_pages <= topk) {  // budget covers every page
        if (blockIdx.x == 0) {
            for (int i = threadIdx.x; i < n_pages; i += blockDim.x)
                s.sel[(int64_t)hx * s.SELCAP + i] = i;
            if (threadIdx.x == 0) s.n_sel[hx] = n_pages;
        }
        return;
    }
    const int n_cand = do_select ? n_pages - 1 : n_pages;
    const int n_chunks = (n_cand + chunk_pages - 1) / chunk_pages;
    if ((int)blockIdx.x >= n_chunks) return;
    const int p0 = blockIdx.x * chunk_pages;
    const int p1 = min(n_cand, p0 + chunk_pages);
    load_group_coeffs<T>(s, q, b, h, w);
    __syncthreads();
    float *row = scores + (int64_t)bh * s.NCAP;
    score_range<T, D>(s, hx, p0, p1, w, row);
    if (!do_select) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) row[n_pages - 1] = -INFINITY;  // pinned
    // last CTA of this head performs the selection
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int ticket = atomicAdd(&counters[bh], 1);
        s_last = (ticket == n_chunks - 1);
        if (s_last) counters[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int i = threadIdx.x; i < n_cand; i += blockDim.x) dyn_keys[i] = score_key(__ldcg(row + i));
    __syncthreads();
    const int kprime = topk - 1;  // n_pages > topk here, so kprime < n_cand
    int32_t *out = s.sel + (int64_t)hx * s.SELCAP;
    if (kprime > 0) block_select<kScoreThreads>(dyn_keys, n_cand, kprime, out);
    if (threadIdx.x == 0) {
        out[kprime] = n_pages - 1;
        s.n_sel[hx] = topk;
    }
}

// standalone select over caller scores: grid n_heads, block kScoreThreads
__global__ void __launch_bounds__(kScoreThreads)
select_topk_kernel(const float *scores, int stride, const int32_t *n_valid, int topk,
                   int pin_last, int32_t *sel_out, int32_t *n_out) {
    extern __shared__ uint32_t dyn_keys[];
    const int hd = blockIdx.x;
    const int n = n_valid[hd];
    int32_t *out = sel_out + (int64_t)hd * topk;
    if (n <= 0) {
        if (threadIdx.x == 0) n_out[hd] = 0;
        return;
    }
    const int budget = min(topk, n);
    const int n_cand = pin_last ? n - 1 : n;
    const int kprime = pin_last ? budget - 1 : budget;
    if (kprime >= n_cand) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = i;
        if (threadIdx.x == 0) n_out[hd] = n;
        return;
    }
    const float *row = scores + (int64_t)hd * stride;
    for (int i = threadIdx.x; i < n_cand; i += blockDim.x) dyn_keys[i] = score_key(row[i]);
    __syncthreads();
    if (kprime > 0) block_select<kScoreThreads>(dyn_keys, n_cand, kprime, out);
    if (threadIdx.x == 0) {
        if (pin_last) out[kprime] = n - 1;
        n_out[hd] = budget;
    }
}

// ---------------------------------------------------------------------------
// launchers

static int score_chunk_pages(int n_pages_max) {
    (void)n_pages_max;
    return 256;
}

template <typename T, int D>
static cudaError_t launch_score_t(const StoreView &s, int layer, const void *q,
                                  const uint8_t *unstable, int period, int force_due, int topk,
                                  int extra, float *scores, int32_t *counters, int do_select,
                                  int batch, cudaStream_t st) {
    const int chunk = score_chunk_pages(s.NCAP);
    dim3 grid((s.NCAP + chunk - 1) / chunk, batch * s.H);
    const size_t smem = do_select ? (size_t)s.NCAP * sizeof(uint32_t) : 0;
    auto kern = score_select_kernel<T, D>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, kScoreThreads, smem, st>>>(s, layer, (const T *)q, unstable, period, force_due,
                                            topk, extra, scores, counters, do_select, chunk);
    return cudaGetLastError();
}

cudaError_t launch_score(const StoreView &s, int dtype, int layer, const void *q,
                         const uint8_t *unstable, int period, int force_due, int topk, int extra,
                         float *scores, int32_t *counters, int do_select, int batch,
                         cudaStream_t st) {
    if (dtype == FC_BF16) {
        if (s.D == 128)
            return launch_score_t<__nv_bfloat16, 128>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, st);
        return launch_score_t<__nv_bfloat16, 64>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, st);
    }
    if (s.D == 128)
        return launch_score_t<float, 128>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, st);
    return launch_score_t<float, 64>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, st);
}

cudaError_t launch_select(const float *scores, int stride, const int32_t *n_valid, int n_heads,
                          int topk, int pin_last, int32_t *sel_out, int32_t *n_out,
                          cudaStream_t st) {
    const size_t smem = (size_t)stride * sizeof(uint32_t);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(select_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    select_topk_kernel<<<n_heads, kScoreThreads, smem, st>>>(scores, stride, n_valid, topk, pin_last,
                                                            sel_out, n_out);
    return cudaGetLastError();
}

}  // namespace fc
