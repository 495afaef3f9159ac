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
// Selection is a block-wide exact threshold search (2 key bits per round) on
// an orderable 32-bit key of the fp32 score (-0.0 == +0.0), ties resolved by
// lowest page index, fused into the last CTA to finish scoring a head
// (threadfence reduction).
#include "attn_warp.cuh"
#include <cub/block/block_scan.cuh>

namespace fc {

// Optional per-CTA timeline for profiling (see fc_debug_attn_trace): [grid][4]
__device__ unsigned long long *g_score_trace = nullptr;
// fused kernel timeline (fc_debug_sa_trace): [grid][4] entry, selection
// visible, attention done, exit
__device__ unsigned long long *g_sa_trace = nullptr;
FC_DEVINL unsigned long long gtimer_s() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kScoreThreads = 256;
#ifndef FC_SCORE_ROUNDS
#define FC_SCORE_ROUNDS 16
#endif
#ifndef FC_SCORE_MINBLOCKS
#define FC_SCORE_MINBLOCKS 2
#endif
constexpr int kRoundsPerIter = FC_SCORE_ROUNDS;   // pages per lane-slot per iteration (MLP)

// ---------------------------------------------------------------------------
// block-wide exact top-K over keys[0..n) in shared memory.
//
// Radix select, MSB digit first, three block-wide passes of 11/11/10 bits on
// an orderable 32-bit key.  Keys live in registers (thread t owns indices
// t + k*NT, so warp w's k-th keys are exactly bit-word w + k*NT/32 of the
// index space).  Each pass: a 2048-bin shared histogram (each warp folds the
// lanes sharing lane 0's digit into one atomic — real scores crowd into few
// top-digit bins), one block scan over the bins, the digit holding the
// kprime-th key.  T = the kprime-th largest key; every key > T is taken plus
// the lowest-index keys == T up to kprime — select_topk's (score desc, index
// asc) order (scoring.py:186).  Selection bits are built per 32-index word
// with ballots and emitted in ascending order after one scan of word counts.
// 0 < kprime < n <= 32*NT.
constexpr int kSelBins = 2048;

constexpr int kSelMaxKptAll = 48;  // = kSelMaxKpt below
// shared scratch of one block_select, declared once for every keys-per-thread
// variant (static shared arrays of separate instantiations would add up)
template <int NT>
struct SelScratch {
    typename cub::BlockScan<int, NT>::TempStorage scan_tmp;
    int hist[kSelBins];
    uint32_t gt_bits[NT * kSelMaxKptAll / 32], eq_bits[NT * kSelMaxKptAll / 32];
    int s_digit, s_above;
    uint32_t s_kmin, s_kmax, s_T;
    int s_rem, s_ncand, s_done;
    uint32_t cand_key[32];
    int cand_idx[32];
    int s_wsum[NT / 32];
};

// One selection scratch per kernel, shared by both selection forms (the
// compact one must not add its own static shared memory: the fused kernels'
// occupancy is set by their shared-memory footprint).
template <int NT>
__device__ __forceinline__ SelScratch<NT> &sel_scratch() {
    __shared__ SelScratch<NT> sc;
    return sc;
}

template <int NT, int KPT>
__device__ void block_select_kpt(const uint32_t *keys, int n, int kprime, int32_t *out, SelScratch<NT> &sc) {
    using Scan = cub::BlockScan<int, NT>;
    constexpr int BPT = kSelBins / NT;  // bins per thread
    constexpr int NWORDS = NT * KPT / 32;
    static_assert(KPT <= kSelMaxKptAll, "scratch sized for kSelMaxKptAll keys per thread");
    auto &scan_tmp = sc.scan_tmp;
    int *hist = sc.hist;
    uint32_t *gt_bits = sc.gt_bits, *eq_bits = sc.eq_bits;
    int &s_digit = sc.s_digit, &s_above = sc.s_above;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t kv[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
        const int i = tid + k * NT;
        kv[k] = i < n ? keys[i] : 0u;  // key 0 never beats a real key (scores are not NaN)
    }
#ifdef FC_SEL_PROFILE
    long long tp[12]; int np_ = 0; tp[np_++] = clock64();
#define FC_SEL_STAMP() tp[np_++] = clock64()
#else
#define FC_SEL_STAMP()
#endif
    uint32_t &s_kmin = sc.s_kmin, &s_kmax = sc.s_kmax, &s_T = sc.s_T;
    int &s_rem = sc.s_rem, &s_ncand = sc.s_ncand, &s_done = sc.s_done;
    uint32_t *cand_key = sc.cand_key;
    int *cand_idx = sc.cand_idx;
    // ---- fast path: one pass of 2048 linear bins over [min key, max key]; the
    // crossing bin of a continuous score distribution holds a handful of keys,
    // ranked exactly by one warp.  Otherwise (ties / skew) the radix passes run.
    {
        uint32_t lo_k = 0xffffffffu, hi_k = 0u;
#pragma unroll
        for (int k = 0; k < KPT; ++k)
            if (tid + k * NT < n) { lo_k = min(lo_k, kv[k]); hi_k = max(hi_k, kv[k]); }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo_k = min(lo_k, __shfl_xor_sync(0xffffffffu, lo_k, o));
            hi_k = max(hi_k, __shfl_xor_sync(0xffffffffu, hi_k, o));
        }
        for (int i = tid; i < kSelBins; i += NT) hist[i] = 0;
        if (tid == 0) { s_kmin = 0xffffffffu; s_kmax = 0u; s_ncand = 0; s_done = 0; }
        __syncthreads();
        if (lane == 0) { atomicMin(&s_kmin, lo_k); atomicMax(&s_kmax, hi_k); }
        __syncthreads();
        // bins linear in the score VALUE (monotone in the key): robust to a few
        // outliers, unlike linear bins in key space
        const float fmin = key_to_float(s_kmin), fmax = key_to_float(s_kmax);
        const float scale = fmax > fmin ? (float)kSelBins / (fmax - fmin) : 0.f;
        auto lbin = [&](uint32_t key) {
            const float b = (key_to_float(key) - fmin) * scale;
            return b >= (float)(kSelBins - 1) ? kSelBins - 1 : (int)b;
        };
#pragma unroll
        for (int k = 0; k < KPT; ++k)
            if (tid + k * NT < n) atomicAdd(&hist[lbin(kv[k])], 1);
        __syncthreads();
        FC_SEL_STAMP();
        int loc[BPT], sum = 0;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            loc[j] = hist[kSelBins - 1 - (tid * BPT + j)];
            sum += loc[j];
        }
        int before, tot;
        Scan(scan_tmp).ExclusiveSum(sum, before, tot);
        int run = before;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            if (run < kprime && run + loc[j] >= kprime) {
                s_digit = kSelBins - 1 - (tid * BPT + j);
                s_above = run;
            }
            run += loc[j];
        }
        __syncthreads();
        FC_SEL_STAMP();
        const int B = s_digit;
        if (hist[B] <= 32) {
#pragma unroll
            for (int k = 0; k < KPT; ++k)
                if (tid + k * NT < n && lbin(kv[k]) == B) {
                    const int slot = atomicAdd(&s_ncand, 1);
                    cand_key[slot] = kv[k];
                    cand_idx[slot] = tid + k * NT;
                }
            __syncthreads();
            if (tid < 32) {
                const int c = s_ncand, need = kprime - s_above;  // 1 <= need <= c
                const uint32_t myk = lane < c ? cand_key[lane] : 0u;
                const int myi = lane < c ? cand_idx[lane] : 0x7fffffff;
                int rank = 0, gt = 0;
                for (int j = 0; j < c; ++j) {
                    const uint32_t kj = __shfl_sync(0xffffffffu, myk, j);
                    const int ij = __shfl_sync(0xffffffffu, myi, j);
                    rank += (kj > myk) || (kj == myk && ij < myi);
                    gt += kj > myk;
                }
                if (lane < c && rank == need - 1) {  // the kprime-th key overall
                    s_T = myk;
                    s_rem = need - gt;                 // keys == T still to take
                    s_done = 1;
                }
            }
        }
        __syncthreads();
        FC_SEL_STAMP();
    }
    uint32_t prefix = 0, mask = 0;
    int remaining = kprime;
    if (s_done) {
        prefix = s_T;
        remaining = s_rem;
    }
#pragma unroll 1
    for (int pass = 0; pass < 3 && !s_done; ++pass) {
        const int shift = pass == 0 ? 21 : pass == 1 ? 10 : 0;
        const uint32_t dmask = pass == 2 ? 0x3ffu : 0x7ffu;
        for (int i = tid; i < kSelBins; i += NT) hist[i] = 0;
        __syncthreads();
        FC_SEL_STAMP();
        {
            // the warp's dominant digit (lane 0's first key) is counted in a
            // register across all KPT keys: one atomic per warp for it, so the
            // crowded top-digit bin sees 8 atomics, not one per key
            const bool v0 = tid < n && (kv[0] & mask) == prefix;
            const int dom = __shfl_sync(0xffffffffu, v0 ? (int)((kv[0] >> shift) & dmask) : -1, 0);
            int dom_cnt = 0;
#pragma unroll
            for (int k = 0; k < KPT; ++k) {
                const bool valid = (tid + k * NT) < n && (kv[k] & mask) == prefix;
                const int d = valid ? (int)((kv[k] >> shift) & dmask) : -1;
                dom_cnt += __popc(__ballot_sync(0xffffffffu, valid && d == dom));
                if (valid && d != dom) atomicAdd(&hist[d], 1);
            }
            if (lane == 0 && dom_cnt) atomicAdd(&hist[dom], dom_cnt);
        }
        __syncthreads();
        FC_SEL_STAMP();
        int loc[BPT], sum = 0;  // descending digits: thread t owns [2047-BPT*t .. 2047-BPT*t-BPT+1]
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            loc[j] = hist[kSelBins - 1 - (tid * BPT + j)];
            sum += loc[j];
        }
        int before, tot;
        Scan(scan_tmp).ExclusiveSum(sum, before, tot);
        int run = before;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            if (run < remaining && run + loc[j] >= remaining) {
                s_digit = kSelBins - 1 - (tid * BPT + j);
                s_above = run;
            }
            run += loc[j];
        }
        __syncthreads();
        prefix |= (uint32_t)s_digit << shift;
        mask |= dmask << shift;
        remaining -= s_above;
        __syncthreads();  // s_digit / hist reuse
        FC_SEL_STAMP();
    }
    const uint32_t T = prefix;
    // selection bit-words: warp w's k-th keys are indices (w + k*NT/32)*32 + lane
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
        const bool inr = (tid + k * NT) < n;
        const unsigned g = __ballot_sync(0xffffffffu, inr && kv[k] > T);
        const unsigned e = __ballot_sync(0xffffffffu, inr && kv[k] == T);
        if (lane == 0) {
            gt_bits[wid + k * (NT / 32)] = g;
            eq_bits[wid + k * (NT / 32)] = e;
        }
    }
    __syncthreads();
    // thread t owns bit-words [t*WPT, t*WPT + WPT) (indices ascending with t)
    constexpr int WPT = (NWORDS + NT - 1) / NT;
    uint32_t eqw[WPT], gtw[WPT];
    int eq_cnt = 0;
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
        const int wd = tid * WPT + u;
        eqw[u] = wd < NWORDS ? eq_bits[wd] : 0u;
        gtw[u] = wd < NWORDS ? gt_bits[wd] : 0u;
        eq_cnt += __popc(eqw[u]);
    }
    int eq_before, dummy;
    Scan(scan_tmp).ExclusiveSum(eq_cnt, eq_before, dummy);
    __syncthreads();
    int take = max(0, min(eq_cnt, remaining - eq_before));  // lowest-index equal keys
    int sel_cnt = 0;
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
        uint32_t e = eqw[u], kept = 0;
        while (take > 0 && e) {
            const uint32_t low = e & (~e + 1u);
            kept |= low;
            e ^= low;
            --take;
        }
        gtw[u] |= kept;
        sel_cnt += __popc(gtw[u]);
    }
    int pos, total_sel;
    Scan(scan_tmp).ExclusiveSum(sel_cnt, pos, total_sel);
#pragma unroll
    for (int u = 0; u < WPT; ++u) {
        uint32_t selw = gtw[u];
        while (selw) {
            const int bit = __ffs(selw) - 1;
            out[pos++] = (tid * WPT + u) * 32 + bit;
            selw &= selw - 1;
        }
    }
    __syncthreads();
    FC_SEL_STAMP();
#ifdef FC_SEL_PROFILE
    if (tid == 0) for (int k = 1; k < np_; ++k) printf("phase %d: %lld cta %d t %lld\n", k, tp[k] - tp[k - 1], (int)blockIdx.x, tp[0]);
#endif
}

// keys per thread by size: up to NT*48 keys (12288 pages at NT = 256, i.e.
// 192k-token heads: config 4's 128k context plus generation)
constexpr int kSelMaxKpt = 48;
template <int NT>
__device__ void block_select(const uint32_t *keys, int n, int kprime, int32_t *out) {
    static_assert(kSelMaxKpt == kSelMaxKptAll, "one scratch size");
    SelScratch<NT> &sc = sel_scratch<NT>();
    if (n <= NT * 8) block_select_kpt<NT, 8>(keys, n, kprime, out, sc);
    else if (n <= NT * 32) block_select_kpt<NT, 32>(keys, n, kprime, out, sc);
    else block_select_kpt<NT, kSelMaxKpt>(keys, n, kprime, out, sc);
}

// Compact form of the same selection for a CTA that runs it alone among
// CTAs streaming pages (the balanced launch's owner): the keys stay in shared
// memory and every pass is a rolled loop over them, so the code is a few
// hundred instructions instead of the unrolled register form's thousands.
// Same result: the kprime largest keys, ties to the lowest index, emitted in
// ascending index order (np.lexsort((arange, -scores))).  The crossing bin
// of the value-linear histogram is ranked exactly when it holds <= 32 keys;
// otherwise (ties / skew) it returns false and the caller runs the unrolled
// block_select (one call site per kernel: a second inlined copy of the
// unrolled form doubles the kernel's code).
template <int NT>
__device__ bool block_select_compact(const uint32_t *keys, int n, int kprime, int32_t *out) {
    SelScratch<NT> &sc = sel_scratch<NT>();
    int *hist = sc.hist, *s_wsum = sc.s_wsum, *cand_idx = sc.cand_idx;
    uint32_t *cand_key = sc.cand_key;
    uint32_t &s_kmin = sc.s_kmin, &s_kmax = sc.s_kmax, &s_T = sc.s_T;
    int &s_digit = sc.s_digit, &s_above = sc.s_above, &s_ncand = sc.s_ncand, &s_rem = sc.s_rem;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    uint32_t lo = 0xffffffffu, hi = 0u;
#pragma unroll 1
    for (int i = tid; i < n; i += NT) { const uint32_t k = keys[i]; lo = min(lo, k); hi = max(hi, k); }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
#pragma unroll 1
    for (int i = tid; i < kSelBins; i += NT) hist[i] = 0;
    if (tid == 0) { s_kmin = 0xffffffffu; s_kmax = 0u; s_ncand = 0; }
    __syncthreads();
    if (lane == 0) { atomicMin(&s_kmin, lo); atomicMax(&s_kmax, hi); }
    __syncthreads();
    const float fmin = key_to_float(s_kmin), fmax = key_to_float(s_kmax);
    const float scale = fmax > fmin ? (float)kSelBins / (fmax - fmin) : 0.f;
    auto lbin = [&](uint32_t key) {
        const float b = (key_to_float(key) - fmin) * scale;
        return b >= (float)(kSelBins - 1) ? kSelBins - 1 : (int)b;
    };
#pragma unroll 1
    for (int i = tid; i < n; i += NT) atomicAdd(&hist[lbin(keys[i])], 1);
    __syncthreads();
    // descending bins: thread t owns bins [kSelBins-1-t*BPT .. -BPT+1]
    constexpr int BPT = kSelBins / NT;
    int sum = 0;
#pragma unroll 1
    for (int j = 0; j < BPT; ++j) sum += hist[kSelBins - 1 - (tid * BPT + j)];
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    int before = x - sum;
#pragma unroll 1
    for (int w = 0; w < wid; ++w) before += s_wsum[w];
    int run = before;
#pragma unroll 1
    for (int j = 0; j < BPT; ++j) {
        const int c = hist[kSelBins - 1 - (tid * BPT + j)];
        if (run < kprime && run + c >= kprime) { s_digit = kSelBins - 1 - (tid * BPT + j); s_above = run; }
        run += c;
    }
    __syncthreads();
    const int B = s_digit;
    if (hist[B] > 32) {  // (ties / skew: the caller runs the general path)
        __syncthreads();
        return false;
    }
#pragma unroll 1
    for (int i = tid; i < n; i += NT)
        if (lbin(keys[i]) == B) {
            const int slot = atomicAdd(&s_ncand, 1);
            cand_key[slot] = keys[i];
            cand_idx[slot] = i;
        }
    __syncthreads();
    if (tid < 32) {
        const int c = s_ncand, need = kprime - s_above;
        const uint32_t myk = lane < c ? cand_key[lane] : 0u;
        const int myi = lane < c ? cand_idx[lane] : 0x7fffffff;
        int rank = 0, gt = 0;
#pragma unroll 1
        for (int j = 0; j < c; ++j) {
            const uint32_t kj = __shfl_sync(0xffffffffu, myk, j);
            const int ij = __shfl_sync(0xffffffffu, myi, j);
            rank += (kj > myk) || (kj == myk && ij < myi);
            gt += kj > myk;
        }
        if (lane < c && rank == need - 1) { s_T = myk; s_rem = need - gt; }
    }
    __syncthreads();
    const uint32_t T = s_T;
    const int rem = s_rem;
    // bit-words of keys > T and == T, 32 indices per word, one warp per word
    const int nw = (n + 31) / 32;  // <= NT * kSelMaxKpt / 32 (n_cand's bound)
    uint32_t *gtb = sc.gt_bits, *eqb = sc.eq_bits;
#pragma unroll 1
    for (int w = wid; w < nw; w += NT / 32) {
        const int i = w * 32 + lane;
        const uint32_t k = i < n ? keys[i] : 0u;
        const unsigned g = __ballot_sync(0xffffffffu, i < n && k > T);
        const unsigned e = __ballot_sync(0xffffffffu, i < n && k == T);
        if (lane == 0) { gtb[w] = g; eqb[w] = e; }
    }
    __syncthreads();
    // thread t owns words [t*WPT, t*WPT + WPT): the lowest-index equal keys
    // are taken first, then every selected index is written in order
    const int WPT = (nw + NT - 1) / NT;
    int eq_cnt = 0;
#pragma unroll 1
    for (int u = 0; u < WPT; ++u) { const int wd = tid * WPT + u; if (wd < nw) eq_cnt += __popc(eqb[wd]); }
    x = eq_cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    __syncthreads();
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    int eq_before = x - eq_cnt;
#pragma unroll 1
    for (int w = 0; w < wid; ++w) eq_before += s_wsum[w];
    int take = max(0, min(eq_cnt, rem - eq_before));
    int sel_cnt = 0;
#pragma unroll 1
    for (int u = 0; u < WPT; ++u) {
        const int wd = tid * WPT + u;
        if (wd >= nw) break;
        uint32_t e = eqb[wd], kept = 0;
        while (take > 0 && e) { const uint32_t low = e & (~e + 1u); kept |= low; e ^= low; --take; }
        gtb[wd] |= kept;
        sel_cnt += __popc(gtb[wd]);
    }
    x = sel_cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int y = __shfl_up_sync(0xffffffffu, x, o); if (lane >= o) x += y; }
    __syncthreads();
    if (lane == 31) s_wsum[wid] = x;
    __syncthreads();
    int pos = x - sel_cnt;
#pragma unroll 1
    for (int w = 0; w < wid; ++w) pos += s_wsum[w];
#pragma unroll 1
    for (int u = 0; u < WPT; ++u) {
        const int wd = tid * WPT + u;
        if (wd >= nw) break;
        uint32_t selw = gtb[wd];
        while (selw) { out[pos++] = wd * 32 + (__ffs(selw) - 1); selw &= selw - 1; }
    }
    __syncthreads();
    return true;
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
// RPI = pages per lane-slot per iteration: the loads a lane keeps in flight.
template <typename T, int D, int RPI = kRoundsPerIter>
__device__ void score_range(const StoreView &s, int hx, int p0, int p1, const float *w,
                            float *scores_row) {
    constexpr int kRoundsPerIter = RPI;
    using Gm = ScoreGeom<T, D>;
    constexpr int kPagesPerIter = Gm::kPagesPerSlot * RPI;
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
    for (int it0 = p0 + warp * kPagesPerIter; it0 < p1; it0 += nwarps * kPagesPerIter) {
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
        // transpose-reduce R values over LPP lanes: log2(R) halving steps, then
        // plain butterflies over the LPP/R lanes that share a round; lane bits
        // then select which round a lane holds.
        static_assert(LPP >= kRoundsPerIter, "rounds per iteration exceed lanes per page");
        constexpr int NSTEP = kRoundsPerIter == 32 ? 5 : kRoundsPerIter == 16 ? 4 : kRoundsPerIter == 8 ? 3
                            : kRoundsPerIter == 4 ? 2 : 1;
        int ridx = 0;
#pragma unroll
        for (int step = 0, dist = LPP / 2, cnt = kRoundsPerIter / 2; step < NSTEP;
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
        for (int dist = LPP / kRoundsPerIter / 2; dist > 0; dist >>= 1)
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], dist);
        if ((cl & (LPP / kRoundsPerIter - 1)) == 0) {
            const int p = it0 + ridx * Gm::kPagesPerSlot + sub;
            if (p < p1) scores_row[p] = v[0];
        }
    }
}

// Scores n consecutive page records starting at rec0 (global memory or, for
// SMEM, a staged copy in shared memory) into out[0, n): score_range's lane
// layout and reduction, so the scores are bit-identical to it.
template <typename T, int D, int RPI, bool SMEM>
__device__ void score_span(const char *rec0, int n, const float *w, float *out) {
    using Gm = ScoreGeom<T, D>;
    constexpr int LPP = Gm::kLanesPerPage, CPL = Gm::kChunksPerLane, EPC = Gm::kElemsPerChunk;
    constexpr int PPI = Gm::kPagesPerSlot * RPI;
    static_assert(LPP >= RPI, "rounds per iteration exceed lanes per page");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
    const int sub = lane / LPP, cl = lane % LPP;
    float coef[CPL][EPC];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < EPC; ++e) coef[c][e] = w[(cl + c * LPP) * EPC + e];
    for (int it0 = warp * PPI; it0 < n; it0 += nwarps * PPI) {
        uint4 raw[RPI][CPL];
#pragma unroll
        for (int r = 0; r < RPI; ++r) {
            const int p = it0 + r * Gm::kPagesPerSlot + sub;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const uint4 *src = reinterpret_cast<const uint4 *>(rec0 + (int64_t)p * Gm::kRecBytes + (cl + c * LPP) * 16);
                if (p < n) raw[r][c] = SMEM ? *src : __ldg(src);
                else raw[r][c] = make_uint4(0, 0, 0, 0);
            }
        }
        float v[RPI];
#pragma unroll
        for (int r = 0; r < RPI; ++r) {
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
        constexpr int NSTEP = RPI == 32 ? 5 : RPI == 16 ? 4 : RPI == 8 ? 3 : RPI == 4 ? 2 : 1;
        int ridx = 0;
#pragma unroll
        for (int step = 0, dist = LPP / 2, cnt = RPI / 2; step < NSTEP; ++step, dist >>= 1, cnt >>= 1) {
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
        for (int dist = LPP / RPI / 2; dist > 0; dist >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], dist);
        if ((cl & (LPP / RPI - 1)) == 0) {
            const int p = it0 + ridx * Gm::kPagesPerSlot + sub;
            if (p < n) out[p] = v[0];
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

// One wave of CTAs over the concatenation of every scored head's candidate
// pages (all pages for do_select = 0; pages [0, n_pages-1) of due heads with
// n_pages > topk for do_select = 1, the last page being pinned).  Each CTA
// takes an equal contiguous range and walks it head segment by head segment;
// for do_select the last CTA to finish a head (threadfence reduction) runs
// the exact selection.  Heads whose budget covers every page are selected
// directly by CTA 0 (all pages).
template <typename T, int D>
__global__ void __launch_bounds__(kScoreThreads, FC_SCORE_MINBLOCKS)
score_select_kernel(StoreView s, int layer, const T *__restrict__ q,
                    const uint8_t *__restrict__ unstable, int period, int force_due,
                    int topk, int extra_tokens, float *scores, int32_t *counters,
                    int do_select, int n_heads, int kv_prefetch) {
    extern __shared__ uint32_t dyn[];  // keys [NCAP] (do_select) | prefix [n_heads+1]
    __shared__ float w[2 * D];
    __shared__ int s_last, s_wsum[kScoreThreads / 32];
    griddep_launch_dependents();
    // kv_prefetch: the previous launch does not write this layer's summaries,
    // selection or seq_len — plan the range and warm L2 before waiting for q
    if (!kv_prefetch) griddep_wait();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long *trace = g_score_trace;
    if (trace && tid == 0) trace[blockIdx.x * 4] = gtimer_s();
    uint32_t *keys = dyn;
    int *prefix = reinterpret_cast<int *>(dyn + (do_select ? s.NCAP : 0));
    const int step = *s.step;

    // ---- candidate counts and prefix over heads
    {
        int carry = 0;
        for (int c0 = 0; c0 < n_heads; c0 += blockDim.x) {
            const int bh = c0 + tid;
            int cnt = 0;
            if (bh < n_heads) {
                const int b = bh / s.H, h = bh % s.H;
                const int n_tok = s.seq_len[b] + extra_tokens;
                const int n_pages = n_tok > 0 ? (n_tok + s.PS - 1) / s.PS : 0;
                if (!do_select) {
                    cnt = n_pages;
                } else if (s.head_due(step, b, unstable[layer * s.H + h], period, force_due)) {
                    if (blockIdx.x == 0 && n_pages > 0) s.count(FC_STAT_SCORE_EVALS, 1);
                    if (n_pages > topk) {
                        cnt = n_pages - 1;
                    } else if (blockIdx.x == 0 && n_pages > 0) {  // budget covers every page
                        const int hx = s.hix(b, layer, h);
                        for (int i = 0; i < n_pages; ++i) s.sel[(int64_t)hx * s.SELCAP + i] = i;
                        s.n_sel[hx] = n_pages;
                    }
                }
            }
            int x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[wid] = x;
            __syncthreads();
            int before = carry, total = 0;
            for (int ww = 0; ww < kScoreThreads / 32; ++ww) {
                if (ww < wid) before += s_wsum[ww];
                total += s_wsum[ww];
            }
            if (bh < n_heads) prefix[bh] = before + x - cnt;
            carry += total;
            __syncthreads();
        }
        if (tid == 0) prefix[n_heads] = carry;
        __syncthreads();
    }
    const int total = prefix[n_heads];
    if (total == 0) return;
    using Gm = ScoreGeom<T, D>;
    constexpr int ALIGN = (kScoreThreads / 32) * Gm::kPagesPerIter;  // one iteration of every warp
    int P = (total + gridDim.x - 1) / gridDim.x;
    P = ((P + ALIGN - 1) / ALIGN) * ALIGN;
    const int start = blockIdx.x * P;
    if (start >= total) {
        if (kv_prefetch) griddep_wait();
        return;
    }
    const int end = min(total, start + P);
    if (kv_prefetch) {
        // warm L2 with the first 64 KiB of this CTA's summaries, then wait for q
        int lo = 0, hi = n_heads - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= start) lo = mid; else hi = mid - 1;
        }
        const int hx0 = s.hix(lo / s.H, layer, lo % s.H);
        const int p0 = start - prefix[lo];
        const int np = min(min(end, prefix[lo + 1]) - start, 65536 / ScoreGeom<T, D>::kRecBytes);
        const char *base = reinterpret_cast<const char *>(s.summ) +
                           ((int64_t)hx0 * s.NCAP + p0) * ScoreGeom<T, D>::kRecBytes;
        const int bytes = np * ScoreGeom<T, D>::kRecBytes;
        for (int off = tid * 4096; off < bytes; off += blockDim.x * 4096)
            bulk_prefetch_l2(base + off, (uint32_t)min(4096, bytes - off));
        griddep_wait();
    }

    int pos = start;
    while (pos < end) {
        int lo = 0, hi = n_heads - 1;  // head containing pos (last with prefix <= pos)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= pos) lo = mid; else hi = mid - 1;
        }
        const int bh = lo;
        const int h_beg = prefix[bh], h_end = prefix[bh + 1];
        const int seg_end = min(end, h_end);
        const int b = bh / s.H, h = bh % s.H;
        const int hx = s.hix(b, layer, h);
        __syncthreads();  // w reuse
        load_group_coeffs<T>(s, q, b, h, w);
        __syncthreads();
        float *row = scores + (int64_t)bh * s.NCAP;
        score_range<T, D>(s, hx, pos - h_beg, seg_end - h_beg, w, row);
        pos = seg_end;
        if (!do_select) continue;
        // ---- the last CTA of this head selects
        const int first_c = h_beg / P, last_c = (h_end - 1) / P;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            const int ticket = atomicAdd(&counters[bh], 1);
            s_last = (ticket == last_c - first_c);
            if (s_last) {
                counters[bh] = 0;
                __threadfence();
            }
        }
        __syncthreads();
        if (trace && tid == 0) trace[blockIdx.x * 4 + 1] = gtimer_s();
        if (!s_last) continue;
        const int n_cand = h_end - h_beg;
        const int n_pages = n_cand + 1;
        // the head's scores (written by every CTA of the head) into keys: 8
        // loads in flight per thread (a load-then-store loop would serialise
        // ~n/256 L2 round trips: ~20 us for a 128k-token head)
        for (int i0 = tid; i0 < n_cand; i0 += blockDim.x * 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = i < n_cand ? __ldcg(row + i) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < n_cand) keys[i] = score_key(v[u]);
            }
        }
        if (tid == 0) row[n_pages - 1] = -INFINITY;  // pinned page: not scored
        __syncthreads();
        const int kprime = topk - 1;  // n_pages > topk, so kprime < n_cand
        int32_t *out = s.sel + (int64_t)hx * s.SELCAP;
        if (kprime > 0) block_select<kScoreThreads>(keys, n_cand, kprime, out);
        if (tid == 0) {
            out[kprime] = n_pages - 1;
            s.n_sel[hx] = topk;
            if (trace) trace[blockIdx.x * 4 + 2] = gtimer_s();
        }
    }
    if (trace && tid == 0) trace[blockIdx.x * 4 + 3] = gtimer_s();
}

// ---------------------------------------------------------------------------
// Head-aligned scoring (batches with at least ~half as many heads as SMs):
// one CTA of 16 warps per due head streams the head's summaries (one
// contiguous [pages][min|max] run) through a ring of 64-page cp.async.bulk
// chunks (~160 KiB in flight), writes the scores straight into shared-memory
// keys and selects right away — no cross-CTA counter, no L2 round trip of the
// scores, and each head's selection overlaps the other heads' streaming.

#ifndef FC_HEAD_WARPS
#define FC_HEAD_WARPS 16
#endif
#ifndef FC_HEAD_CHUNK_PAGES
#define FC_HEAD_CHUNK_PAGES 64
#endif
#ifndef FC_HEAD_LAST_REFILL
#define FC_HEAD_LAST_REFILL 0
#endif
#ifndef FC_HEAD_RING_KB
#define FC_HEAD_RING_KB 160
#endif
constexpr int kHeadScoreWarps = FC_HEAD_WARPS;
#ifndef FC_SCORE_MODE_DEFAULT
#define FC_SCORE_MODE_DEFAULT -1
#endif
static int g_score_mode = FC_SCORE_MODE_DEFAULT;  // -1 auto, 0 balanced, 1 head-aligned (test hook)
static int g_score_ctas_per_sm = 0;  // balanced kernel: CTAs per SM (0: as many as fit)
constexpr int kHeadChunkPages = FC_HEAD_CHUNK_PAGES;

template <typename T, int D, int NWS = kHeadScoreWarps>
struct HeadScoreGeom {
    using Gm = ScoreGeom<T, D>;
    static constexpr int kChunkBytes = kHeadChunkPages * Gm::kRecBytes;
    static constexpr int kStages = (FC_HEAD_RING_KB * 1024) / kChunkBytes > 2 ? (FC_HEAD_RING_KB * 1024) / kChunkBytes : 2;
    static constexpr int kRounds = kHeadChunkPages / (NWS * Gm::kPagesPerSlot);  // per warp per chunk
};

// shared bytes before the fp32 q of the fused kernel: max(scoring ring + keys,
// attention ring / merge scratch)
template <typename T, int D, int NST, int NWA>
__host__ __device__ constexpr size_t score_attend_ring_bytes(int ncap) {
    return (size_t)HeadScoreGeom<T, D>::kStages * HeadScoreGeom<T, D>::kChunkBytes + (size_t)ncap * 4 >
                   (size_t)NWA * NST * AttnGeom<T, D>::kPageBytes
               ? (((size_t)HeadScoreGeom<T, D>::kStages * HeadScoreGeom<T, D>::kChunkBytes + (size_t)ncap * 4 + 127) &
                  ~(size_t)127)
               : (size_t)NWA * NST * AttnGeom<T, D>::kPageBytes;
}

// Streaming half of the head-aligned scoring: rank `rank` of the S CTAs
// scoring head bh streams candidate pages [n_cand*rank/S, n_cand*(rank+1)/S)
// of the head's summaries and writes their keys into keys_dst (the keys array
// of the CTA that selects: its own, or rank 0's through DSMEM) and the scores
// row.  Every thread of the CTA calls it.  Returns 0 (head not due / empty),
// 1 (the budget covers every page: rank 0 wrote the selection) or 2 (keys
// written: the selecting CTA runs score_head_select on n_cand keys).  Waits
// for the previous launch (PDL) on every path.  dsm: ring [NS][chunk] | keys.
template <typename T, int D, int NWS = kHeadScoreWarps>
__device__ int score_head_stream(const StoreView &s, int layer, const T *__restrict__ q,
                                 const uint8_t *__restrict__ unstable, int period, int force_due, int topk,
                                 int extra_tokens, float *scores, int kv_prefetch, char *dsm, uint64_t *full,
                                 uint64_t *empty, int *s_rel, float *w, int bh, int S, int rank,
                                 uint32_t *keys_dst, int &n_cand_out, bool in_cluster = false) {
    // in a cluster the caller arrived on the cluster barrier at entry; wait on
    // it before the first write into another CTA's shared memory (a peer may
    // not have started yet) — and on every other way out
    auto cluster_wait = [&]() {
        if (in_cluster) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    };
    using Gm = ScoreGeom<T, D>;
    using HG = HeadScoreGeom<T, D, NWS>;
    constexpr int NW = NWS, NS = HG::kStages, R = HG::kRounds;
    constexpr int LPP = Gm::kLanesPerPage, CPL = Gm::kChunksPerLane, EPC = Gm::kElemsPerChunk;
    static_assert(R >= 1 && R <= LPP, "chunk geometry");
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned long long *trace = g_score_trace;  // [grid][4]: entry, copies issued, streamed, selected
    if (trace && tid == 0) trace[blockIdx.x * 4] = gtimer_s();
    if (!kv_prefetch) griddep_wait();
    const int b = bh / s.H, h = bh % s.H;
    const bool due = s.head_due(*s.step, b, unstable[layer * s.H + h], period, force_due);
    const int n_tok = s.seq_len[b] + extra_tokens;
    const int n_pages = n_tok > 0 ? (n_tok + s.PS - 1) / s.PS : 0;
    const int hx = s.hix(b, layer, h);
    if (due && n_pages > 0 && rank == 0 && tid == 0) s.count(FC_STAT_SCORE_EVALS, 1);
    if (!due || n_pages == 0) {
        if (kv_prefetch) griddep_wait();
        cluster_wait();
        return 0;
    }
    int32_t *out = s.sel + (int64_t)hx * s.SELCAP;
    if (n_pages <= topk) {  // budget covers every page
        if (kv_prefetch) griddep_wait();
        if (rank == 0) {
            for (int i = tid; i < n_pages; i += blockDim.x) out[i] = i;
            if (tid == 0) s.n_sel[hx] = n_pages;
        }
        cluster_wait();
        return 1;
    }
    const int n_cand_all = n_pages - 1;  // the last page is pinned
    n_cand_out = n_cand_all;
    const int c0 = (int)((int64_t)n_cand_all * rank / S);
    const int n_cand = (int)((int64_t)n_cand_all * (rank + 1) / S) - c0;  // this rank's candidates
    const int n_chunks = (n_cand + kHeadChunkPages - 1) / kHeadChunkPages;
    char *ring = dsm;
    uint32_t *keys = keys_dst + c0;
    const char *base = reinterpret_cast<const char *>(s.summ) + ((int64_t)hx * s.NCAP + c0) * Gm::kRecBytes;
    if (tid == 0) {
        // every consuming thread arrives on `empty` (its own reads precede its
        // arrival; a per-warp arrival after __syncwarp is ordered the same way
        // but racecheck only credits the arriving thread)
        for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NW * 32); s_rel[i] = 0; }
        fence_mbar_init();
        for (int c = 0; c < min(NS, n_chunks); ++c) {
            const uint32_t bytes = min(kHeadChunkPages, n_cand - c * kHeadChunkPages) * Gm::kRecBytes;
            mbar_arrive_expect_tx(&full[c], bytes);
            bulk_g2s(ring + (size_t)c * HG::kChunkBytes, base + (int64_t)c * HG::kChunkBytes, bytes, &full[c]);
        }
    }
    if (kv_prefetch) griddep_wait();  // q comes from the previous launch
    if (trace && tid == 0) trace[blockIdx.x * 4 + 1] = gtimer_s();  // (released)
    load_group_coeffs<T>(s, q, b, h, w);
    __syncthreads();
    const int sub = lane / LPP, cl = lane % LPP;
    float coef[CPL][EPC];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int e = 0; e < EPC; ++e) coef[c][e] = w[(cl + c * LPP) * EPC + e];
    float *srow = scores + (int64_t)bh * s.NCAP + c0;
    cluster_wait();  // every CTA of the cluster has started: keys_dst is valid
    for (int c = 0; c < n_chunks; ++c) {
        const int stg = c % NS;
        mbar_wait(&full[stg], (c / NS) & 1);
        const char *chunk = ring + (size_t)stg * HG::kChunkBytes;
        const int cp = min(kHeadChunkPages, n_cand - c * kHeadChunkPages);
        float v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int p = (wid * R + r) * Gm::kPagesPerSlot + sub;  // page within the chunk
            float acc = 0.f;
            if (p < cp) {
#pragma unroll
                for (int cc = 0; cc < CPL; ++cc) {
                    const uint4 raw = *reinterpret_cast<const uint4 *>(chunk + p * Gm::kRecBytes + (cl + cc * LPP) * 16);
#ifdef FC_SCORE_SKIP_MATH  // profiling variant: the ring without the dot products
                    acc += __uint_as_float(raw.x & 0x3f000000u);
#else
                    float f[EPC];
                    chunk_to_f<T>(raw, f);
#pragma unroll
                    for (int e = 0; e < EPC; ++e) acc = fmaf(f[e], coef[cc][e], acc);
#endif
                }
            }
            v[r] = acc;
        }
        __syncwarp();
#if FC_HEAD_LAST_REFILL
        // the last warp to release the stage refills it (nobody blocks on it)
        if (lane == 0) {
            __threadfence_block();
            const bool last = atomicAdd(&s_rel[stg], 1) == NW - 1;
            if (last && c + NS < n_chunks) {
                s_rel[stg] = 0;
                fence_proxy_async_smem();
                const int cn = c + NS;
                const uint32_t bytes = min(kHeadChunkPages, n_cand - cn * kHeadChunkPages) * Gm::kRecBytes;
                mbar_arrive_expect_tx(&full[stg], bytes);
                bulk_g2s(ring + (size_t)stg * HG::kChunkBytes, base + (int64_t)cn * HG::kChunkBytes, bytes, &full[stg]);
            }
        }
#else
        mbar_arrive(&empty[stg]);  // this thread is done reading the stage
#endif
        // transpose-reduce R values over LPP lanes
        int ridx = 0;
#pragma unroll
        for (int dist = LPP / 2, cnt = R / 2; cnt >= 1; dist >>= 1, cnt >>= 1) {
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
        for (int dist = LPP / R / 2; dist > 0; dist >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], dist);
        if ((cl & (LPP / R - 1)) == 0) {
            const int p = (wid * R + ridx) * Gm::kPagesPerSlot + sub;
            if (p < cp) {
                const int gp = c * kHeadChunkPages + p;
                keys[gp] = score_key(v[0]);
                srow[gp] = v[0];
            }
        }
        // refill this stage once every warp has released it
        if (!FC_HEAD_LAST_REFILL && tid == 0 && c + NS < n_chunks) {
            mbar_wait(&empty[stg], (c / NS) & 1);
            fence_proxy_async_smem();
            const int cn = c + NS;
            const uint32_t bytes = min(kHeadChunkPages, n_cand - cn * kHeadChunkPages) * Gm::kRecBytes;
            mbar_arrive_expect_tx(&full[stg], bytes);
            bulk_g2s(ring + (size_t)stg * HG::kChunkBytes, base + (int64_t)cn * HG::kChunkBytes, bytes, &full[stg]);
        }
    }
    if (tid == 0 && rank == 0) scores[(int64_t)bh * s.NCAP + n_pages - 1] = -INFINITY;  // pinned: not scored
    __syncthreads();
    if (trace && tid == 0) trace[blockIdx.x * 4 + 2] = gtimer_s();
    return 2;
}

// Selecting half: the kprime = topk-1 best of the n_cand keys, then the
// pinned last page (select_topk, scoring.py:164-193).  Every thread of the
// selecting CTA calls it.
template <int NT>
__device__ void score_head_select(const StoreView &s, const uint32_t *keys, int n_cand, int topk, int hx,
                                  bool compact = false) {
    int32_t *out = s.sel + (int64_t)hx * s.SELCAP;
    const int kprime = topk - 1;  // n_pages > topk, so kprime < n_cand
    if (kprime > 0) {
        // beyond 8 keys per thread the unrolled register form's code (16 / 32
        // / 48 keys per thread) outgrows the instruction cache: the rolled
        // form is faster in a launch (config 4, 128k: 74.5 -> 70.4 us per
        // scored layer); up to 8 the unrolled form wins (config 2: 52.8 vs
        // 53.9 us)
        if (!(compact && n_cand > NT * 8 && block_select_compact<NT>(keys, n_cand, kprime, out)))
            block_select<NT>(keys, n_cand, kprime, out);
    }
    if (threadIdx.x == 0) {
        out[kprime] = n_cand;  // = n_pages - 1
        s.n_sel[hx] = topk;
        unsigned long long *trace = g_score_trace;
        if (trace) trace[blockIdx.x * 4 + 3] = gtimer_s();
    }
}

// Body of the head-aligned scoring for head blockIdx.x (one CTA per head):
// stream, then select.  Returns after the selection is in s.sel / s.n_sel
// (or at once for a head that is not due).
template <typename T, int D, int NWS = kHeadScoreWarps>
__device__ void score_head_body(const StoreView &s, int layer, const T *__restrict__ q,
                                const uint8_t *__restrict__ unstable, int period, int force_due, int topk,
                                int extra_tokens, float *scores, int kv_prefetch, char *dsm, uint64_t *full,
                                uint64_t *empty, int *s_rel, float *w) {
    using HG = HeadScoreGeom<T, D, NWS>;
    uint32_t *keys = reinterpret_cast<uint32_t *>(dsm + (size_t)HG::kStages * HG::kChunkBytes);
    int n_cand = 0;
    const int st = score_head_stream<T, D, NWS>(s, layer, q, unstable, period, force_due, topk, extra_tokens,
                                                  scores, kv_prefetch, dsm, full, empty, s_rel, w, blockIdx.x, 1,
                                                  0, keys, n_cand);
    if (st == 2) {
        const int b = blockIdx.x / s.H, h = blockIdx.x % s.H;
        score_head_select<NWS * 32>(s, keys, n_cand, topk, s.hix(b, layer, h));
    }
}


template <typename T, int D>
__global__ void __launch_bounds__(kHeadScoreWarps * 32, 1)
score_head_kernel(StoreView s, int layer, const T *__restrict__ q, const uint8_t *__restrict__ unstable,
                  int period, int force_due, int topk, int extra_tokens, float *scores, int kv_prefetch) {
    extern __shared__ __align__(128) char dsm[];  // ring [NS][chunk] | keys [NCAP]
    __shared__ __align__(8) uint64_t full[HeadScoreGeom<T, D>::kStages], empty[HeadScoreGeom<T, D>::kStages];
    __shared__ int s_rel[HeadScoreGeom<T, D>::kStages];
    __shared__ float w[2 * D];
    griddep_launch_dependents();
    score_head_body<T, D>(s, layer, q, unstable, period, force_due, topk, extra_tokens, scores, kv_prefetch,
                          dsm, full, empty, s_rel, w);
}

// Ring stages of a head in a scoring launch: a head that is not scored
// (score_head_stream status != 2) streams through one stage fewer (a.bal_nst
// < 0, the default; 0: all stages), so the heads that score and select first
// take a larger share of the saturated HBM for their attention.
template <int NST>
FC_DEVINL int unscored_stages(const AttnArgs &a, int st) {
    if (st == 2 || a.bal_nst == 0) return NST;
    const int want = a.bal_nst < 0 ? NST - 1 : a.bal_nst;
    return want > 0 && want < NST ? want : NST;
}

// Fused scoring + attention of one head per CTA (layers whose heads are
// scored this step): the selection never leaves the CTA's view before its
// pages stream — no grid-wide wait between scoring and attention, no second
// launch, no selection -> table round trip through another kernel.  NWS warps
// score (16 for bf16, as the head-aligned scoring kernel); then warps
// NWA..NWS-1 hand their registers over (setmaxnreg: the scoring phase fits
// 128 registers per thread, the attention state needs ~210) and leave, and
// warps 0..NWA-1 attend exactly as attn_kernel (attend_head_cta); the ring
// reuses the scoring ring / keys.  Same results as fc_score_select followed
// by fc_sparse_decode (the attention reads the selection just written).
// Next-layer summary warm-up (AttnArgs::pf_cap).  With unstable heads spread
// over every layer, a plain step's fused launch mixes scored heads (summaries
// + pages: 2 MB at config 2) and unscored ones (pages: 1 MB); one CTA per
// head, so the scored CTAs are the layer's critical path while the others sit
// idle after their pages.  Those idle CTAs here pull the NEXT layer's due
// summaries into L2 (cp.async.bulk.prefetch.L2), so that layer's scored CTAs
// stream their summaries at L2 rather than HBM rate.  Nothing a launch writes
// is in those records except the appended page, which is never scored (the
// last page is pinned), so the warm-up reads final data.  The next layer of
// layer L-1 is layer 0 of the next step (step + 1).  `ord` / `n_pf` = this
// CTA's ordinal among the launch's prefetching CTAs / their number; every
// prefetching CTA takes an equal share of the due pages.  Called by one warp
// (all lanes): lanes cover rows, so the per-row state (each row's own step,
// its reload hold) is read once per row and in parallel.
static constexpr int64_t kSummaryPrefetchCap = 48ll << 20;  // L2 = 126 MB: leave room for the pages streaming by
static int64_t g_summary_prefetch_cap = kSummaryPrefetchCap;

// heads of row b due in layer l at global step step0 (bit h), for rows held
// waiting for a reload none; unstable heads every step, all at the boundary
FC_DEVINL uint32_t row_due_mask(const StoreView &s, int step0, int b, int l, const uint8_t *__restrict__ unstable,
                               int period, int force_due) {
    const uint32_t all = s.H >= 32 ? 0xffffffffu : (1u << s.H) - 1;
    if (force_due) return all;
    if (s.hold_mode(b) == FC_HOLD_WAIT) return 0;
    if (s.boundary(step0, b, period)) return all;
    uint32_t m = 0;
    for (int h = 0; h < s.H && h < 32; ++h) m |= unstable[l * s.H + h] ? (1u << h) : 0u;
    return m;
}

template <typename T, int D>
__device__ void prefetch_next_summaries(const StoreView &s, int layer, const uint8_t *__restrict__ unstable,
                                        int period, int topk, int extra_tokens, int batch, int ord, int n_pf,
                                        int64_t cap) {
    using Gm = ScoreGeom<T, D>;
    const int lane = threadIdx.x & 31;
    int nl = layer + 1, step = *s.step;
    if (nl == s.L) { nl = 0; ++step; }
    // candidate pages of the due heads, per row (lanes), then over rows
    int64_t total = 0;
    for (int b0 = 0; b0 < batch; b0 += 32) {
        const int b = b0 + lane;
        int64_t mine = 0;
        if (b < batch) {
            const int n_tok = s.seq_len[b] + extra_tokens;
            const int np = n_tok > 0 ? (n_tok + s.PS - 1) / s.PS : 0;
            if (np > topk) mine = (int64_t)(np - 1) * __popc(row_due_mask(s, step, b, nl, unstable, period, 0));
        }
        for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
        total += mine;
    }
    if (total == 0 || total * Gm::kRecBytes > cap) return;
    if (lane != 0) return;
    int64_t lo = total * ord / n_pf;
    const int64_t hi = total * (ord + 1) / n_pf;
    int64_t base = 0;
    for (int b = 0; b < batch && lo < hi; ++b) {
        const int n_tok = s.seq_len[b] + extra_tokens;
        const int np = n_tok > 0 ? (n_tok + s.PS - 1) / s.PS : 0;
        if (np <= topk) continue;
        const int cand = np - 1;
        const uint32_t due = row_due_mask(s, step, b, nl, unstable, period, 0);
        if (base + (int64_t)cand * __popc(due) <= lo) {  // the whole row is before this share
            base += (int64_t)cand * __popc(due);
            continue;
        }
        for (int h = 0; h < s.H && lo < hi; ++h) {
            if (!((due >> h) & 1u)) continue;
            if (lo < base + cand) {
                const int p0 = (int)(lo - base);
                const int p1 = (int)(hi - base < cand ? hi - base : cand);
                const char *src = reinterpret_cast<const char *>(s.summ) +
                                  ((int64_t)s.hix(b, nl, h) * s.NCAP + p0) * Gm::kRecBytes;
                for (int64_t off = 0, n = (int64_t)(p1 - p0) * Gm::kRecBytes; off < n; off += 65536)
                    bulk_prefetch_l2(src + off, (uint32_t)(n - off < 65536 ? n - off : 65536));
                lo = base + p1;
            }
            base += cand;
        }
    }
}

template <int NWS, int NWA>
struct RegSplit {  // registers per thread after the hand-over (multiples of 8)
    static constexpr int kBase = 65536 / (NWS * 32) > 255 ? 255 : 65536 / (NWS * 32);
    static constexpr int kLow = 24;
    static constexpr int kHigh = ((65536 - (NWS - NWA) * 32 * kLow) / (NWA * 32)) / 8 * 8 > 248
                                     ? 248 : ((65536 - (NWS - NWA) * 32 * kLow) / (NWA * 32)) / 8 * 8;
};

template <typename T, int D, int NST, int NWA, int NWS, bool CL>
__global__ void __launch_bounds__(NWS * 32, 1)
score_attend_kernel(StoreView s, int layer, const T *__restrict__ q, const uint8_t *__restrict__ unstable,
                    int period, int force_due, int topk, int extra_tokens, float *scores, int kv_prefetch,
                    AttnArgs a, int S_arg) {
    // CL = false: one CTA per head (S = 1, no cluster code compiled in: the
    // attention phase keeps its registers); CL = true: a cluster of S_arg
    const int S = CL ? S_arg : 1;
    static_assert(NWS >= NWA && NWS % 4 == 0 && NWA % 4 == 0, "whole warpgroups");
    namespace cg = cooperative_groups;
    using HG = HeadScoreGeom<T, D, NWS>;
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t full[HG::kStages], empty[HG::kStages];
    __shared__ int s_rel[HG::kStages];
    __shared__ float w[2 * D];
    __shared__ __align__(8) uint64_t abars[NWA * NST];
    __shared__ float s_wm[NWA][16], s_wl[NWA][16];
    griddep_launch_dependents();
    unsigned long long *satr = g_sa_trace;
    if (satr && threadIdx.x == 0) satr[blockIdx.x * 4] = gtimer_s();
    // S CTAs (a cluster) per head: every rank scores its share of the pages
    // into rank 0's keys (DSMEM), rank 0 selects, every rank attends its
    // share of the selection, rank 0 merges the ranks' states (DSMEM)
    int bh = blockIdx.x / S, rank = blockIdx.x % S, Sh = S;  // head, rank and CTAs on it
    if constexpr (CL) {
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // waited in the stream
        if (a.cta_map) {  // mixed clusters (host-written map, read before the PDL wait)
            const int e = a.cta_map[blockIdx.x];
            bool idle = e < 0;
            if (!idle) {
                bh = e & ~(1 << 30);
                if (e & (1 << 30)) { Sh = 1; rank = 0; }
                if (bh >= a.map_heads) { set_error(s.err, FC_ERR_RUN_RANGE); idle = true; }
            }
            if (idle) {  // every cluster barrier of the kernel, no work
                griddep_wait();
                asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
                cg::this_cluster().sync();
                cg::this_cluster().sync();
                if (a.out == nullptr) return;
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
                return;
            }
        }
    }
    const int b = bh / s.H, h = bh % s.H, hx = s.hix(b, layer, h);
    uint32_t *keys = reinterpret_cast<uint32_t *>(dsm + (size_t)HG::kStages * HG::kChunkBytes);
    uint32_t *keys_dst = keys;
    if constexpr (CL) {
        if (Sh > 1) keys_dst = cg::this_cluster().map_shared_rank(keys, 0);
    }
    int n_cand = 0;
    const int st = score_head_stream<T, D, NWS>(s, layer, q, unstable, period, force_due, topk, extra_tokens,
                                                  scores, kv_prefetch, dsm, full, empty, s_rel, w, bh, Sh, rank,
                                                  keys_dst, n_cand, CL);
    if constexpr (CL) cg::this_cluster().sync();  // every rank's keys are in rank 0
    if (st == 2 && rank == 0)
        score_head_select<NWS * 32>(s, keys, n_cand, topk, hx, a.compact_select != 0);
    if constexpr (CL) cg::this_cluster().sync();  // the selection (global) is visible to every rank
    else __syncthreads();                         // selection written by this CTA; scoring smem free
    if (a.out == nullptr) return;                 // scoring only (fc_score_select at small batches)
    const bool attends = (int)(threadIdx.x >> 5) < NWA;
    if constexpr (NWS > NWA) {
        if (!attends) {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(RegSplit<NWS, NWA>::kLow));
            if constexpr (CL) {  // the cluster's two merge barriers, in as few registers as possible
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            }
            return;
        }
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(RegSplit<NWS, NWA>::kHigh));
    }
    float *s_q = reinterpret_cast<float *>(dsm + score_attend_ring_bytes<T, D, NST, NWA>(s.NCAP));
    // the CTA's state for the cluster merge lives past the attention scratch
    float *cstate = reinterpret_cast<float *>(dsm) + (size_t)NWA * s.G * D;
    if constexpr (!CL) {
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 1] = gtimer_s();
        attend_head_cta<T, D, NST, NWA>(s, a, bh, dsm, abars, s_wm, s_wl, s_q, 1, 1, 0, nullptr,
                                        unscored_stages<NST>(a, st));
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 2] = gtimer_s();
        if (a.pf_cap > 0 && threadIdx.x < 32) {
            // the heads not due share the prefetch: this one's ordinal among
            // them (lanes over rows: each row's due mask read once)
            const int step = *s.step, lane = threadIdx.x;
            const int batch = gridDim.x / s.H;
            const uint32_t all = s.H >= 32 ? 0xffffffffu : (1u << s.H) - 1;
            if (!((row_due_mask(s, step, b, layer, unstable, period, force_due) >> h) & 1u)) {
                int nnd = 0, before = 0;
                for (int b0 = 0; b0 < batch; b0 += 32) {
                    const int bb = b0 + lane;
                    int nd = 0, bef = 0;
                    if (bb < batch) {
                        const uint32_t notdue = ~row_due_mask(s, step, bb, layer, unstable, period, force_due) & all;
                        nd = __popc(notdue);
                        bef = bb < b ? nd : (bb == b ? __popc(notdue & ((1u << h) - 1)) : 0);
                    }
                    for (int o = 16; o > 0; o >>= 1) {
                        nd += __shfl_xor_sync(0xffffffffu, nd, o);
                        bef += __shfl_xor_sync(0xffffffffu, bef, o);
                    }
                    nnd += nd;
                    before += bef;
                }
                prefetch_next_summaries<T, D>(s, layer, unstable, period, topk, extra_tokens, batch,
                                              before, nnd, a.pf_cap);
            }
        }
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 3] = gtimer_s();
    } else {
        // (only attending warps get here when NWS > NWA)
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 1] = gtimer_s();
        const int n_att = attend_head_cta<T, D, NST, NWA>(s, a, bh, dsm, abars, s_wm, s_wl, s_q, 1, Sh, rank,
                                                          Sh > 1 ? cstate : nullptr, unscored_stages<NST>(a, st));
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 2] = gtimer_s();
        // every rank's state written
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (Sh > 1 && rank == 0 && n_att > 0) merge_head_cluster<T, D>(s, a, bh, cstate, Sh, NWA * 32);
        // rank 0 done reading every rank's shared memory
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (satr && threadIdx.x == 0) satr[blockIdx.x * 4 + 3] = gtimer_s();
    }
}

// ---------------------------------------------------------------------------
// A load that is re-issued on every call (other CTAs of the launch update the word).
FC_DEVINL int ld_relaxed_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Balanced fused score + select + attend (fc_score_attend_balanced).
//
// The head-aligned fused kernel gives each head ONE CTA for its scoring and
// its attention.  When only some heads of a layer are due (a plain step with
// the unstable heads spread over the layers: 2 of 8 KV heads at config 2), a
// scored CTA streams its summaries (1 MB at 32k) and then its pages (1 MB)
// while an unscored CTA streams only its pages: the layer takes the time of
// the scored CTA, ~2x the unscored one (45 vs 25 us, scripts/spread_probe.py).
// Here every CTA of a one-wave grid (max(heads, SMs) CTAs, all co-resident)
// first scores an equal share of the concatenation of the due heads'
// candidate pages (score_range, as score_select_kernel), publishing each
// finished head segment with a release counter; then CTA i < heads attends
// head i: an unscored head at once, a scored head after its owner CTA (CTA
// i itself) has waited for every segment of its scores, selected from them
// and written the selection (the keys alias the attention ring).  The
// scoring work is spread over every SM, so the due summaries stream at the
// whole GPU's rate instead of one SM's.  Results: the same per-page scores
// and selections as fc_score_select's balanced kernel (same score_range),
// the same attention as fc_sparse_decode (attend_head_cta).
// Requires every CTA co-resident (the owners wait on the others): the
// launcher checks the occupancy.  bf16 only (8 warps score and attend).
#ifndef FC_BAL_BULK_SCORES
#define FC_BAL_BULK_SCORES 1
#endif
#ifndef FC_BAL_ROUNDS
#define FC_BAL_ROUNDS 32
#endif
template <typename T, int D, int NST, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
score_attend_bal_kernel(StoreView s, int layer, const T *__restrict__ q, const uint8_t *__restrict__ unstable,
                        int period, int force_due, int topk, int extra_tokens, float *scores, int32_t *counters,
                        int n_heads, int kv_prefetch, AttnArgs a) {
    static_assert(NW * 32 == kScoreThreads, "the scoring phase runs on kScoreThreads threads");
    using Gm = ScoreGeom<T, D>;
    constexpr size_t kRing = (size_t)NW * NST * AttnGeom<T, D>::kPageBytes;
    // dynamic: ring [NW][NST][page] (the selecting CTA's keys alias it) | prefix [n_heads + 1]
    extern __shared__ __align__(128) char dsm[];
    __shared__ float w[2 * D];
    __shared__ int s_wsum[NW];
    __shared__ __align__(8) uint64_t abars[NW * NST];
    __shared__ float s_wm[NW][16], s_wl[NW][16];
    __shared__ __align__(8) uint64_t stage_bar;
    __shared__ __align__(8) uint64_t keys_bar;
    griddep_launch_dependents();
    unsigned long long *satr = g_sa_trace;
    if (satr && threadIdx.x == 0) satr[blockIdx.x * 8] = gtimer_s();
    // without kv_prefetch the previous launch may write this layer's
    // selection / seq_len: wait before reading anything
    if (!kv_prefetch) griddep_wait();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int *prefix = reinterpret_cast<int *>(dsm + kRing);
    uint32_t *keys = reinterpret_cast<uint32_t *>(dsm);
    const int step = *s.step;
    auto is_due = [&](int bh) {
        return s.head_due(step, bh / s.H, unstable[layer * s.H + bh % s.H], period, force_due);
    };
    auto pages_of = [&](int b) {
        const int n_tok = s.seq_len[b] + extra_tokens;
        return n_tok > 0 ? (n_tok + s.PS - 1) / s.PS : 0;
    };
    // ---- candidate counts of the due heads (the last page is pinned) and their prefix
    {
        int carry = 0;
        for (int c0 = 0; c0 < n_heads; c0 += blockDim.x) {
            const int bh = c0 + tid;
            int cnt = 0;
            if (bh < n_heads && is_due(bh)) {
                const int np = pages_of(bh / s.H);
                cnt = np > topk ? np - 1 : 0;
            }
            int x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[wid] = x;
            __syncthreads();
            int before = carry, tot = 0;
            for (int ww = 0; ww < NW; ++ww) {
                if (ww < wid) before += s_wsum[ww];
                tot += s_wsum[ww];
            }
            if (bh < n_heads) prefix[bh] = before + x - cnt;
            carry += tot;
            __syncthreads();
        }
        if (tid == 0) prefix[n_heads] = carry;
        __syncthreads();
    }
    const int total = prefix[n_heads];
    // 32 (d = 128): 16 KiB of loads in flight per warp; at most the lanes of a page
    constexpr int RPI = FC_BAL_ROUNDS < Gm::kLanesPerPage ? FC_BAL_ROUNDS : Gm::kLanesPerPage;
    int P = (total + gridDim.x - 1) / gridDim.x;
    P = (P + 31) & ~31;  // equal shares over every CTA (a coarser grain leaves CTAs idle)
    const int start = min(total, (int)blockIdx.x * P), end = min(total, start + P);
    // head containing candidate position pos (the last with prefix <= pos)
    auto head_of = [&](int pos) {
        int lo = 0, hi = n_heads - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (prefix[mid] <= pos) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    auto rec_of = [&](int bh, int page) {
        return reinterpret_cast<const char *>(s.summ) +
               ((int64_t)s.hix(bh / s.H, layer, bh % s.H) * s.NCAP + page) * Gm::kRecBytes;
    };
    // Stage the head of this CTA's share into shared memory (the ring, idle
    // until phase 2) with bulk copies issued BEFORE waiting for the previous
    // launch: the summaries of this layer are final (the previous launch
    // appends into its own layer, and a due head's last page is never
    // scored), only q is not.  The rest of the share is read from global.
    const int staged_end = min(end, start + (int)(kRing / Gm::kRecBytes));
    if (tid == 0) {
        mbar_init(&stage_bar, 1);
        fence_mbar_init();
        if (start < staged_end) {
            mbar_arrive_expect_tx(&stage_bar, (uint32_t)(staged_end - start) * Gm::kRecBytes);
            for (int pos = start; pos < staged_end;) {
                const int bh = head_of(pos), seg = min(staged_end, prefix[bh + 1]);
                const char *src = rec_of(bh, pos - prefix[bh]);
                char *dst = dsm + (size_t)(pos - start) * Gm::kRecBytes;
                for (int64_t off = 0, nb = (int64_t)(seg - pos) * Gm::kRecBytes; off < nb; off += 65536)
                    bulk_g2s(dst + off, src + off, (uint32_t)(nb - off < 65536 ? nb - off : 65536), &stage_bar);
                pos = seg;
            }
        }
    }
    if (satr && tid == 0) satr[blockIdx.x * 8 + 1] = gtimer_s();
    if (kv_prefetch) griddep_wait();  // q comes from the previous launch
    if (satr && tid == 0) satr[blockIdx.x * 8 + 2] = gtimer_s();
    // ---- phase 1: this CTA's share of the due pages; each finished head segment is published
    bool landed = false;
    for (int pos = start; pos < end;) {
        const int bh = head_of(pos), h_beg = prefix[bh], seg_end = min(end, prefix[bh + 1]);
        const int b = bh / s.H, h = bh % s.H;
        __syncthreads();  // w reuse
        load_group_coeffs<T>(s, q, b, h, w);
        __syncthreads();
        float *row = scores + (int64_t)bh * s.NCAP - h_beg;  // indexed by candidate position
        const int mid = max(pos, min(seg_end, staged_end));  // [pos, mid) staged, [mid, seg_end) from global
        if (pos < mid) {
            if (!landed) {
                mbar_wait(&stage_bar, 0);
                landed = true;
                if (satr && tid == 0) satr[blockIdx.x * 8 + 3] = gtimer_s();
            }
            score_span<T, D, RPI, true>(dsm + (size_t)(pos - start) * Gm::kRecBytes, mid - pos, w, row + pos);
        }
        if (mid < seg_end) score_span<T, D, RPI, false>(rec_of(bh, mid - h_beg), seg_end - mid, w, row + mid);
        pos = seg_end;
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicAdd(&counters[bh], 1);
        }
    }
    if (satr && threadIdx.x == 0) satr[blockIdx.x * 8 + 4] = gtimer_s();
    // Chunked attention of the scored heads (a.bal_flags != nullptr): the
    // attended pages of a head with candidates are cut into NC chunks
    // (attend_head_cta's rank r of NC).  Its owner claims chunks of it once
    // its selection is out; every CTA with no work of its own left (the CTAs
    // beyond one per head after scoring, unscored owners after their head,
    // owners after their chunks) claims chunks of any scored head whose
    // selection is out.  Chunk states go to global memory; the CTA finishing
    // a head's last chunk merges them.  Per-head words: ready (= epoch + 1
    // once the selection is out; the owner zeroes claim / done before), claim
    // (next chunk; over-claims are harmless), done.  The epoch is constant
    // within a launch and advanced by the last CTA to exit, so a word left by
    // an earlier launch never reads as ready (the next launch reads it after
    // griddepcontrol.wait, i.e. after this launch completed).
    const bool steal = a.bal_flags != nullptr;
    const int NC = steal ? a.max_splits : 1;
    const int GD = s.G * D + 32;
    int32_t *ready = steal ? a.bal_flags : nullptr;
    int32_t *claim = steal ? a.bal_flags + n_heads : nullptr;
    int32_t *done = steal ? a.bal_flags + 2 * n_heads : nullptr;
    int32_t *glob = steal ? a.bal_flags + 4 * n_heads : nullptr;  // [0] epoch, [1] CTAs exited
    __shared__ int s_epoch, s_pick, s_pend, s_chunk, s_merge;
    if (steal) {
        if (tid == 0) s_epoch = ld_relaxed_gpu(glob);
        __syncthreads();
    }
    const int epoch1 = steal ? s_epoch + 1 : 0;
    // attend chunk c of scored head hb; the CTA finishing its last chunk merges
    auto run_chunk = [&](int hb, int c) {
        float *st0 = a.bal_state + (int64_t)hb * kBalMaxSplit * GD;
        const int n_att = attend_head_cta<T, D, NST, NW>(s, a, hb, dsm, abars, s_wm, s_wl, nullptr, 1, NC, c,
                                                         st0 + (int64_t)c * GD);
        __syncthreads();  // every thread's state written
        if (tid == 0) {
            int old;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(done + hb) : "memory");
            s_merge = old == NC - 1;
        }
        __syncthreads();
        if (s_merge && n_att > 0) merge_head_global<T, D>(s, a, hb, st0, NC, blockDim.x);
        __syncthreads();  // s_merge read by every thread before it is rewritten
    };
    // claim chunks of any scored head until none is left or pending
    auto help = [&]() {
        const int off = (int)(((int64_t)blockIdx.x * n_heads) / gridDim.x);
        while (true) {
            if (tid == 0) { s_pick = INT_MAX; s_pend = 0; }
            __syncthreads();
            for (int x = tid; x < n_heads; x += blockDim.x) {
                if (prefix[x + 1] <= prefix[x]) continue;
                if (ld_relaxed_gpu(ready + x) != epoch1) s_pend = 1;
                else if (ld_relaxed_gpu(claim + x) < NC) atomicMin(&s_pick, (x - off + n_heads) % n_heads);
            }
            __syncthreads();
            const int pick = s_pick, pend = s_pend;
            __syncthreads();  // read by every thread before tid 0 rewrites them
            if (satr && tid == 0 && (int)blockIdx.x >= n_heads) {  // (profiling: the help loop's state)
                satr[blockIdx.x * 8 + 5] += 1;
                satr[blockIdx.x * 8 + 6] = pick;
                satr[blockIdx.x * 8 + 1] = pend;
            }
            if (pick == INT_MAX) {
                if (!pend || !a.bal_wait) break;
                if (tid == 0) __nanosleep(200);
                continue;
            }
            const int hb = (pick + off) % n_heads;
            if (tid == 0) {
                int r;
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(r) : "l"(ready + hb) : "memory");
                s_chunk = atomicAdd(claim + hb, 1);
            }
            __syncthreads();
            const int c = s_chunk;
            if (c < NC) run_chunk(hb, c);
        }
    };
    // every CTA passes here once on its way out
    auto leave = [&]() {
        __syncthreads();
        if (tid == 0) {
            const int old = atomicAdd(glob + 1, 1);
            if (old == (int)gridDim.x - 1) {  // last CTA of the launch: advance the epoch
                glob[1] = 0;
                __threadfence();
                glob[0] = epoch1;
            }
        }
    };
    if ((int)blockIdx.x >= n_heads) {
        if (steal) {
            help();
            leave();
        }
        return;
    }
    // ---- phase 2: CTA bh owns head bh
    const int bh = blockIdx.x, b = bh / s.H, h = bh % s.H, hx = s.hix(b, layer, h);
    const bool chunked = steal && prefix[bh + 1] > prefix[bh];
    const int n_pages = pages_of(b);
    if (is_due(bh) && n_pages > 0) {
        if (tid == 0) s.count(FC_STAT_SCORE_EVALS, 1);
        int32_t *out = s.sel + (int64_t)hx * s.SELCAP;
        if (n_pages <= topk) {  // budget covers every page
            for (int i = tid; i < n_pages; i += blockDim.x) out[i] = i;
            if (tid == 0) s.n_sel[hx] = n_pages;
        } else {
            const int h_beg = prefix[bh], h_end = prefix[bh + 1], n_cand = h_end - h_beg;
            const int expect = (h_end - 1) / P - h_beg / P + 1;  // CTAs that scored a segment of it
            float *row = scores + (int64_t)bh * s.NCAP;
            if (tid == 0) {
                int got;
                while (true) {
                    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(got) : "l"(counters + bh) : "memory");
                    if (got >= expect) break;
                    __nanosleep(64);
                }
                if (satr) satr[blockIdx.x * 8 + 5] = gtimer_s();
                counters[bh] = 0;  // self-resetting for the next launch
                row[n_pages - 1] = -INFINITY;  // pinned page: not scored
            }
#if FC_BAL_BULK_SCORES
            // the score row in ONE bulk copy into shared memory (one request
            // under the launch's full HBM load instead of 2047 loads), then
            // converted to keys
            float *raw = reinterpret_cast<float *>(keys + ((2 * s.NCAP + 3) & ~3));  // 16-byte aligned, past the keys
            const uintptr_t src0 = reinterpret_cast<uintptr_t>(row) & ~uintptr_t(15);
            const int off = (int)((reinterpret_cast<uintptr_t>(row) - src0) / 4);
            if (tid == 0) {
                mbar_init(&keys_bar, 1);
                fence_mbar_init();
                asm volatile("fence.proxy.async.global;" ::: "memory");  // the scores are generic-proxy writes
                const uint32_t nb = (uint32_t)(((off + n_cand) * 4 + 15) & ~15);
                mbar_arrive_expect_tx(&keys_bar, nb);
                bulk_g2s(raw, reinterpret_cast<const void *>(src0), nb, &keys_bar);
            }
            __syncthreads();
            mbar_wait(&keys_bar, 0);
            for (int i = tid; i < n_cand; i += blockDim.x) keys[i] = score_key(raw[off + i]);
#else
            __syncthreads();
            for (int i0 = tid; i0 < n_cand; i0 += blockDim.x * 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    v[u] = i < n_cand ? __ldcg(row + i) : 0.f;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < n_cand) keys[i] = score_key(v[u]);
                }
            }
#endif
            __syncthreads();
            const int kprime = topk - 1;  // n_pages > topk, so kprime < n_cand
            if (satr && tid == 0) satr[blockIdx.x * 8 + 1] = gtimer_s();  // (owner: keys in smem)
            // the selection is emitted into shared memory (the ring past the
            // keys) and copied out coalesced
            int32_t *sel_s = reinterpret_cast<int32_t *>(keys + s.NCAP);
#ifndef FC_BAL_UNROLLED_SELECT
            if (kprime > 0 && !block_select_compact<kScoreThreads>(keys, n_cand, kprime, sel_s))
                block_select<kScoreThreads>(keys, n_cand, kprime, sel_s);
#else
            if (kprime > 0) block_select<kScoreThreads>(keys, n_cand, kprime, sel_s);
#endif
            if (satr && tid == 0) satr[blockIdx.x * 8 + 3] = gtimer_s();  // (owner: selected)
            __syncthreads();
            for (int i = tid; i < kprime; i += blockDim.x) out[i] = sel_s[i];
            if (tid == 0) {
                out[kprime] = n_pages - 1;
                s.n_sel[hx] = topk;
            }
        }
        __syncthreads();  // the selection is written; the keys are dead (the ring reuses them)
    }
    if (chunked && tid == 0) {
        // the selection is out (the barrier above orders every thread's writes
        // before this release, which is cumulative): chunks may be claimed
        claim[bh] = 0;
        done[bh] = 0;
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ready + bh), "r"(epoch1) : "memory");
    }
    if (satr && threadIdx.x == 0) satr[blockIdx.x * 8 + 6] = gtimer_s();
    if (!chunked) {
        // a head that is not scored streams through fewer stages (a.bal_nst;
        // default one fewer): with fewer of its pages in flight it takes a
        // smaller share of the saturated HBM, and the scored heads, which
        // start their attention ~8 us later, a larger one (config 2: spread
        // mask 12.80k -> 12.94k, staggered phases 12.23k -> 12.51k tokens/s;
        // one stage: slower)
        const int want = a.bal_nst < 0 ? NST - 1 : a.bal_nst;
        const int nst = (want > 0 && want < NST && !is_due(bh)) ? want : NST;
        attend_head_cta<T, D, NST, NW>(s, a, bh, dsm, abars, s_wm, s_wl, nullptr, 1, 1, 0, nullptr, nst);
    } else {
        while (true) {  // this head's chunks first
            if (tid == 0) s_chunk = atomicAdd(claim + bh, 1);
            __syncthreads();
            const int c = s_chunk;
            __syncthreads();
            if (c >= NC) break;
            run_chunk(bh, c);
        }
    }
    if (steal) {
        help();
        leave();
    }
    if (satr && threadIdx.x == 0) satr[blockIdx.x * 8 + 7] = gtimer_s();
}

template <typename T, int D, int NST, int NW>
static size_t score_attend_bal_smem(int n_heads) {
    return (size_t)NW * NST * AttnGeom<T, D>::kPageBytes + (size_t)(n_heads + 1) * sizeof(int);
}

// CTAs of the balanced fused launch for this batch, 0 if it does not fit
// (every CTA must be co-resident; the selection keys must fit in the ring)
template <typename T, int D, int NST, int NW>
static int score_attend_bal_grid_t(const StoreView &s, int batch) {
    const int n_heads = batch * s.H;
    // (the ring holds the owner's keys and its selection during the select)
    // (the ring holds the owner's keys, the select's scratch and the score row's bulk copy)
    const size_t need = (size_t)max(3 * s.NCAP + 12, s.NCAP + s.SELCAP) * 4;
    if (n_heads < 1 || need > (size_t)NW * NST * AttnGeom<T, D>::kPageBytes) return 0;
    if (s.NCAP > kScoreThreads * kSelMaxKpt) return 0;
    auto k = score_attend_bal_kernel<T, D, NST, NW>;
    const size_t smem = score_attend_bal_smem<T, D, NST, NW>(n_heads);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0, dev = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NW * 32, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = n_heads > sms ? n_heads : sms;
    return occ >= 1 && grid <= occ * sms ? grid : 0;
}

int score_attend_balanced_grid(const StoreView &s, int dtype, int batch) {
    if (dtype != FC_BF16) return 0;
    return s.D == 128 ? score_attend_bal_grid_t<__nv_bfloat16, 128, 3, 8>(s, batch)
                      : score_attend_bal_grid_t<__nv_bfloat16, 64, 6, 8>(s, batch);
}

template <typename T, int D, int NST, int NW>
static cudaError_t launch_score_attend_bal_t(const StoreView &s, int layer, const void *q, const uint8_t *unstable,
                                             int period, int force_due, int topk, int extra, float *scores,
                                             int32_t *counters, int batch, int kv_prefetch, const AttnArgs &a,
                                             cudaStream_t st) {
    const int grid = score_attend_bal_grid_t<T, D, NST, NW>(s, batch);
    if (grid < 1) return cudaErrorInvalidConfiguration;
    const int n_heads = batch * s.H;
    return launch_pdl(score_attend_bal_kernel<T, D, NST, NW>, dim3(grid), dim3(NW * 32),
                      score_attend_bal_smem<T, D, NST, NW>(n_heads), st, s, layer, (const T *)q, unstable, period,
                      force_due, topk, extra, scores, counters, n_heads, kv_prefetch, a);
}

cudaError_t launch_score_attend_balanced(const StoreView &s, int dtype, int layer, const void *q,
                                         const uint8_t *unstable, int period, int force_due, int topk, int extra,
                                         float *scores, int32_t *counters, int batch, int kv_prefetch,
                                         const AttnArgs &a, cudaStream_t st) {
    if (dtype != FC_BF16) return cudaErrorInvalidConfiguration;
    if (s.D == 128)
        return launch_score_attend_bal_t<__nv_bfloat16, 128, 3, 8>(
            s, layer, q, unstable, period, force_due, topk, extra, scores, counters, batch, kv_prefetch, a, st);
    return launch_score_attend_bal_t<__nv_bfloat16, 64, 6, 8>(s, layer, q, unstable, period, force_due, topk, extra,
                                                              scores, counters, batch, kv_prefetch, a, st);
}

// Exact select over float64 scores (the per-call select_topk API on the
// reference's own float64 scores, scoring.py:164-193): the rank of each page
// among all — a higher score, or an equal score at a lower index, ranks
// first (np.lexsort((arange, -scores))) — counted against every other page
// (n <= 12288: at most 1.5e8 comparisons), then the pages of rank < kprime
// (and the pinned last page) compacted in ascending index order by one CTA.
// No rounding of the scores, so no ties that float64 does not have.
__global__ void __launch_bounds__(256)
rank_f64_kernel(const double *__restrict__ scores, int n, int kprime, int pin_last, uint8_t *keep) {
    __shared__ double tile[1024];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int nc = pin_last ? n - 1 : n;  // candidates (the last page is pinned)
    const double si = i < nc ? scores[i] : 0.0;
    int rank = 0;
    for (int t0 = 0; t0 < nc; t0 += 1024) {
        __syncthreads();
        for (int j = threadIdx.x; j < 1024 && t0 + j < nc; j += blockDim.x) tile[j] = scores[t0 + j];
        __syncthreads();
        const int m = min(1024, nc - t0);
        if (i < nc)
            for (int j = 0; j < m; ++j) {
                const double sj = tile[j];
                rank += (sj > si) || (sj == si && t0 + j < i);
            }
    }
    if (i < n) keep[i] = (i < nc) ? (rank < kprime) : 1;
}

__global__ void __launch_bounds__(1024) compact_keep_kernel(const uint8_t *keep, int n, int32_t *out, int32_t *n_out) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    int carry = 0;
    for (int c0 = 0; c0 < n; c0 += 1024) {
        const int i = c0 + threadIdx.x;
        const int f = i < n ? keep[i] : 0;
        int pos, tot;
        Scan(tmp).ExclusiveSum(f, pos, tot);
        if (f) out[carry + pos] = i;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_out = carry;
}

cudaError_t launch_select_f64(const double *scores, int n, int topk, int pin_last, uint8_t *keep, int32_t *out,
                              int32_t *n_out, cudaStream_t st) {
    const int kprime = pin_last ? topk - 1 : topk;  // (k >= n: every page)
    rank_f64_kernel<<<(n + 255) / 256, 256, 0, st>>>(scores, n, kprime, pin_last, keep);
    compact_keep_kernel<<<1, 1024, 0, st>>>(keep, n, out, n_out);
    return cudaGetLastError();
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
    for (int i0 = threadIdx.x; i0 < n_cand; i0 += blockDim.x * 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            v[u] = i < n_cand ? row[i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x;
            if (i < n_cand) dyn_keys[i] = score_key(v[u]);
        }
    }
    __syncthreads();
    if (kprime > 0) block_select<kScoreThreads>(dyn_keys, n_cand, kprime, out);
    if (threadIdx.x == 0) {
        if (pin_last) out[kprime] = n - 1;
        n_out[hd] = budget;
    }
}

// ---------------------------------------------------------------------------
// launchers

template <typename T, int D>
static cudaError_t launch_score_t(const StoreView &s, int layer, const void *q,
                                  const uint8_t *unstable, int period, int force_due, int topk,
                                  int extra, float *scores, int32_t *counters, int do_select,
                                  int batch, int kv_prefetch, cudaStream_t st) {
    const int n_heads = batch * s.H;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const bool head_mode = g_score_mode < 0 ? 2 * n_heads >= sms : g_score_mode == 1;
    using HG = HeadScoreGeom<T, D>;
    const size_t hsmem = (size_t)HG::kStages * HG::kChunkBytes + (size_t)s.NCAP * sizeof(uint32_t);
    auto hk = score_head_kernel<T, D>;
    static size_t hstatic = SIZE_MAX;
    if (hstatic == SIZE_MAX) {
        cudaFuncAttributes fa{};
        if (cudaFuncGetAttributes(&fa, hk) != cudaSuccess) return cudaGetLastError();
        hstatic = fa.sharedSizeBytes;
    }
    if (do_select && head_mode && hsmem + hstatic <= 227 * 1024) {  // head-aligned: one CTA per head
        static size_t hcached = 0;
        if (hcached != hsmem) {
            if (cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsmem) != cudaSuccess)
                return cudaGetLastError();
            hcached = hsmem;
        }
        return launch_pdl(hk, dim3(n_heads), dim3(kHeadScoreWarps * 32), hsmem, st, s, layer, (const T *)q,
                          unstable, period, force_due, topk, extra, scores, kv_prefetch);
    }
    const size_t smem = (do_select ? (size_t)s.NCAP * sizeof(uint32_t) : 0) + (size_t)(n_heads + 1) * sizeof(int);
    auto kern = score_select_kernel<T, D>;
    static size_t cached_smem = (size_t)-1;
    static int grid = 0, cached_cps = -1;
    if (cached_smem != smem || cached_cps != g_score_ctas_per_sm) {  // one full wave at the occupancy this smem allows
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        // the SM's largest shared-memory split: the attention launch that
        // follows (PDL) can then co-reside with this one
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        int occ = 0, dev = 0, sms = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kScoreThreads, smem);
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_score_ctas_per_sm > 0 && g_score_ctas_per_sm < occ) occ = g_score_ctas_per_sm;
        grid = (occ < 1 ? 1 : occ) * sms;
        cached_smem = smem;
        cached_cps = g_score_ctas_per_sm;
    }
    return launch_pdl(kern, dim3(grid), dim3(kScoreThreads), smem, st, s, layer, (const T *)q, unstable,
                      period, force_due, topk, extra, scores, counters, do_select, n_heads, kv_prefetch);
}

cudaError_t launch_score(const StoreView &s, int dtype, int layer, const void *q,
                         const uint8_t *unstable, int period, int force_due, int topk, int extra,
                         float *scores, int32_t *counters, int do_select, int batch,
                         int kv_prefetch, cudaStream_t st) {
    if (dtype == FC_BF16) {
        if (s.D == 128)
            return launch_score_t<__nv_bfloat16, 128>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, kv_prefetch, st);
        return launch_score_t<__nv_bfloat16, 64>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, kv_prefetch, st);
    }
    if (s.D == 128)
        return launch_score_t<float, 128>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, kv_prefetch, st);
    return launch_score_t<float, 64>(s, layer, q, unstable, period, force_due, topk, extra, scores, counters, do_select, batch, kv_prefetch, st);
}

// fused score + attend: head-aligned only (one CTA per head)
template <typename T, int D, int NST, int NWA, int NWS = NWA>
static size_t score_attend_smem(const StoreView &s) {
    return score_attend_ring_bytes<T, D, NST, NWA>(s.NCAP) + (sizeof(T) == 4 ? (size_t)s.G * D * sizeof(float) : 0);
}

template <typename T, int D, int NST, int NWA, int NWS, bool CL = false>
static int score_attend_fits_t(const StoreView &s) {
    auto k = score_attend_kernel<T, D, NST, NWA, NWS, CL>;
    const size_t smem = score_attend_smem<T, D, NST, NWA, NWS>(s);
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NWS * 32, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return occ >= 1;
}

// CTAs per head: 1 when the batch fills the GPU with heads (the head-aligned
// rule); otherwise the largest power of two <= 16 that keeps one wave with
// every cluster co-resident.  0: does not fit.
template <typename T, int D, int NST, int NWA, int NWS>
static int score_attend_split_t(const StoreView &s, int batch) {
    if (!score_attend_fits_t<T, D, NST, NWA, NWS, false>(s) || !score_attend_fits_t<T, D, NST, NWA, NWS, true>(s))
        return 0;
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    const int heads = batch * s.H;
    if (g_score_mode == 1 || (g_score_mode < 0 && 2 * heads >= sms)) return 1;
    if (g_score_mode == 0) return 0;
    auto k = score_attend_kernel<T, D, NST, NWA, NWS, true>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int best = 0;
    for (int S = 2; S <= max_cluster() && heads * S <= sms; S *= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(heads * S);
        cfg.blockDim = dim3(NWS * 32);
        cfg.dynamicSmemBytes = score_attend_smem<T, D, NST, NWA, NWS>(s);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (clusters >= heads) best = S;
    }
    return best;
}

template <typename T, int D, int NST, int NWA, int NWS>
static cudaError_t launch_score_attend_t(const StoreView &s, int layer, const void *q, const uint8_t *unstable,
                                         int period, int force_due, int topk, int extra, float *scores,
                                         int batch, int kv_prefetch, const AttnArgs &a, cudaStream_t st) {
    const int S = score_attend_split_t<T, D, NST, NWA, NWS>(s, batch);
    if (S < 1) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch * s.H * S);
    cfg.blockDim = dim3(NWS * 32);
    cfg.dynamicSmemBytes = score_attend_smem<T, D, NST, NWA, NWS>(s);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = S;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = S > 1 ? 2 : 1;
    static const int compact = std::getenv("FC_SA_COMPACT") ? std::atoi(std::getenv("FC_SA_COMPACT")) : 1;
    if (S > 1) {
        AttnArgs ac = a;
        ac.compact_select = compact;
        return cudaLaunchKernelEx(&cfg, score_attend_kernel<T, D, NST, NWA, NWS, true>, s, layer, (const T *)q,
                                  unstable, period, force_due, topk, extra, scores, kv_prefetch, ac, S);
    }
    AttnArgs a1 = a;
    a1.pf_cap = g_summary_prefetch_cap;
    a1.compact_select = compact;
    return cudaLaunchKernelEx(&cfg, score_attend_kernel<T, D, NST, NWA, NWS, false>, s, layer, (const T *)q, unstable,
                              period, force_due, topk, extra, scores, kv_prefetch, a1, 1);
}

// mixed clusters (fc_score_attend_map): n_ctas CTAs in clusters of S (a
// cluster of S fits on the device)
template <typename T, int D, int NST, int NWA, int NWS>
static int score_attend_map_fits_t(const StoreView &s, int n_ctas, int S) {
    if (S < 2 || S > 16 || n_ctas < S || n_ctas % S) return 0;
    if (!score_attend_fits_t<T, D, NST, NWA, NWS, true>(s)) return 0;
    auto k = score_attend_kernel<T, D, NST, NWA, NWS, true>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_ctas);
    cfg.blockDim = dim3(NWS * 32);
    cfg.dynamicSmemBytes = score_attend_smem<T, D, NST, NWA, NWS>(s);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&clusters, k, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    // clusters never wait on each other: a grid beyond one wave runs in waves
    return clusters >= 1;
}

template <typename T, int D, int NST, int NWA, int NWS>
static cudaError_t launch_score_attend_map_t(const StoreView &s, int layer, const void *q, const uint8_t *unstable,
                                             int period, int force_due, int topk, int extra, float *scores,
                                             int kv_prefetch, const AttnArgs &a, int n_ctas, int S,
                                             cudaStream_t st) {
    if (!score_attend_map_fits_t<T, D, NST, NWA, NWS>(s, n_ctas, S)) return cudaErrorInvalidConfiguration;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_ctas);
    cfg.blockDim = dim3(NWS * 32);
    cfg.dynamicSmemBytes = score_attend_smem<T, D, NST, NWA, NWS>(s);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = S;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, score_attend_kernel<T, D, NST, NWA, NWS, true>, s, layer, (const T *)q,
                              unstable, period, force_due, topk, extra, scores, kv_prefetch, a, S);
}

#ifndef FC_SA_SCORE_WARPS
#define FC_SA_SCORE_WARPS 16
#endif
// attention ring stages / attending warps of the fused kernel, bf16 d = 128
#ifndef FC_SA_NST128
#define FC_SA_NST128 3
#endif
#ifndef FC_SA_NWA128
#define FC_SA_NWA128 8
#endif
#define FC_SA_DISPATCH(dtype, D, CALL)                                                  \
    ((dtype) == FC_BF16 ? ((D) == 128 ? CALL(__nv_bfloat16, 128, FC_SA_NST128, FC_SA_NWA128, FC_SA_SCORE_WARPS) \
                                      : CALL(__nv_bfloat16, 64, 6, 8, FC_SA_SCORE_WARPS))               \
                        : ((D) == 128 ? CALL(float, 128, 3, 4, 4) : CALL(float, 64, 6, 4, 4)))

// CTAs per head of the fused kernel for this batch (0: not supported)
int score_attend_supported(const StoreView &s, int dtype, int batch) {
    if (batch < 1) return 0;
#define FC_SAF(T, DD, N, W, WS) score_attend_split_t<T, DD, N, W, WS>(s, batch)
    return FC_SA_DISPATCH(dtype, s.D, FC_SAF);
#undef FC_SAF
}

cudaError_t launch_score_attend(const StoreView &s, int dtype, int layer, const void *q, const uint8_t *unstable,
                                int period, int force_due, int topk, int extra, float *scores, int batch,
                                int kv_prefetch, const AttnArgs &a, cudaStream_t st) {
#define FC_SAL(T, DD, N, W, WS) \
    launch_score_attend_t<T, DD, N, W, WS>(s, layer, q, unstable, period, force_due, topk, extra, scores, batch, kv_prefetch, a, st)
    return FC_SA_DISPATCH(dtype, s.D, FC_SAL);
#undef FC_SAL
}

int score_attend_map_fits(const StoreView &s, int dtype, int n_ctas, int S) {
#define FC_SAM(T, DD, N, W, WS) score_attend_map_fits_t<T, DD, N, W, WS>(s, n_ctas, S)
    return FC_SA_DISPATCH(dtype, s.D, FC_SAM);
#undef FC_SAM
}

cudaError_t launch_score_attend_map(const StoreView &s, int dtype, int layer, const void *q, const uint8_t *unstable,
                                    int period, int force_due, int topk, int extra, float *scores, int kv_prefetch,
                                    const AttnArgs &a, int n_ctas, int S, cudaStream_t st) {
#define FC_SAML(T, DD, N, W, WS) \
    launch_score_attend_map_t<T, DD, N, W, WS>(s, layer, q, unstable, period, force_due, topk, extra, scores, kv_prefetch, a, n_ctas, S, st)
    return FC_SA_DISPATCH(dtype, s.D, FC_SAML);
#undef FC_SAML
}

void set_score_mode(int m) { g_score_mode = m; }
void set_score_ctas_per_sm(int n) { g_score_ctas_per_sm = n; }
void set_summary_prefetch_cap(int64_t bytes) { g_summary_prefetch_cap = bytes < 0 ? kSummaryPrefetchCap : bytes; }

cudaError_t set_sa_trace(void *p) {
    return cudaMemcpyToSymbol(g_sa_trace, &p, sizeof(p));
}

cudaError_t set_score_trace(void *p) {
    return cudaMemcpyToSymbol(g_score_trace, &p, sizeof(p));
}

cudaError_t launch_select(const float *scores, int stride, const int32_t *n_valid, int n_heads,
                          int topk, int pin_last, int32_t *sel_out, int32_t *n_out,
                          cudaStream_t st) {
    const size_t smem = (size_t)stride * sizeof(uint32_t);
    static bool configured = false;
    if (!configured) {  // keys up to 12288 (48 KiB) on top of the static histogram / bit words
        cudaFuncSetAttribute(select_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        configured = true;
    }
    select_topk_kernel<<<n_heads, kScoreThreads, smem, st>>>(scores, stride, n_valid, topk, pin_last,
                                                            sel_out, n_out);
    return cudaGetLastError();
}

}  // namespace fc
