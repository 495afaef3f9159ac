// sparse_decode.cu — subsystem (3): GQA paged sparse decode attention over the
// selected pages, split-K across pages with the combine fused into the last
// CTA of each head.
//
// Reference semantics: _attend / dense_decode / sparse_decode
// (attention.py:67-111): softmax(q·Kᵀ/√d)·V with max subtraction over the
// tokens of the selected pages in ascending page order; a selected page that
// is not resident (null block) is a residency violation (:101-105).  For
// stable heads between reranks the attended set is the last selection plus
// the pages appended since (simulator.py:416-420,512) — here derived on the
// fly as sel[0..n_sel) ∪ (max(sel), n_pages).
//
// Data path (HBM-bound, ~4 flop/B at G=4): each warp owns a private ring of
// NST page buffers filled by cp.async.bulk (TMA 1-D, one 8 KiB copy per bf16
// page: K rows then V rows, contiguous in the block) completing on an
// mbarrier; the page lands in shared memory already XOR-swizzled (see
// page_elem_offset) so ldmatrix is bank-conflict-free.  bf16: q·Kᵀ and P·V on
// the legacy tensor path (mma.sync m16n8k16, query rows padded to 16), online
// softmax in registers with exp2.  fp32: CUDA-core FFMA path (correctness
// mode, 1e-5 parity).  Warps merge through shared memory; splits merge in the
// last CTA of the head (threadfence reduction) — no second launch.
#include "launchers.cuh"
#include "attn_warp.cuh"
#include <cooperative_groups.h>
#include <type_traits>

namespace fc {

constexpr int kMaxClusterCtas = 16;

// Optional per-CTA timeline (globaltimer ns) for profiling: [grid][4] =
// entry, first load issued, main loop done, exit.  Null in production.
__device__ unsigned long long *g_attn_trace = nullptr;

FC_DEVINL unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// one page as FC_PAGE_SPLIT bulk copies on the same mbarrier (tx counted once)
#ifndef FC_PAGE_SPLIT
#define FC_PAGE_SPLIT 1
#endif
#ifndef FC_L2_PREFETCH
#define FC_L2_PREFETCH 0   // pages ahead of the ring warmed into L2 (0 = off)
#endif
FC_DEVINL void bulk_page(char *dst, const char *src, uint32_t bytes, uint64_t *bar) {
    constexpr int NS = FC_PAGE_SPLIT;
#pragma unroll
    for (int k = 0; k < NS; ++k)
        bulk_g2s(dst + k * (bytes / NS), src + k * (bytes / NS), bytes / NS, bar);
}

// One head per cluster of S CTAs (S = 1: a plain CTA).  The head's attended
// pages are cut into S*NW equal contiguous ranges, one per warp; a warp
// streams its pages through a private ring of NST cp.async.bulk stages (one
// copy of the whole page, K then V, completing on an mbarrier) and keeps one
// online-softmax state.  At the end the warps merge through shared memory and
// the S CTAs of the cluster merge through distributed shared memory into
// rank 0, which writes the output — no partials in global memory, no second
// pass.  The warp that stages the head's last page first writes the new
// token into it (fused append).
template <typename T, int D, int NST, int NW>
__global__ void __launch_bounds__(NW * 32)
attn_kernel(StoreView s, AttnArgs a, int S) {
    using Gm = AttnGeom<T, D>;
    // dynamic: ring [NW][NST][page] | (fp32) q [G][D] | cta state [G][D] + m,l [2][16]
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ float s_wm[NW][16], s_wl[NW][16];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = s.G;
    unsigned long long *trace = g_attn_trace;
    const unsigned long long t_entry = trace ? gtimer() : 0ull;
    griddep_launch_dependents();  // let the next launch get scheduled early (PDL)
    // Without kv_prefetch the selection / table / seq_len may come from the
    // previous launch: wait for it.  With kv_prefetch the caller guarantees
    // they do not, so pages are resolved and their loads issued while the
    // previous kernel drains; only q and the new token wait.  A head the
    // preceding scoring launch does not select this step (early_unstable)
    // reads nothing that launch writes: it runs without waiting at all.
    bool early = false;
    if (a.early_unstable != nullptr) {  // (the head is not due: head_due, spelled out lazily)
        const int eb = (blockIdx.x / S) / s.H;
        const int m = s.hold_mode(eb);
        if (m == FC_HOLD_WAIT) early = true;
        else if (!a.early_unstable[a.layer * s.H + (blockIdx.x / S) % s.H])
            early = m == FC_HOLD_RESUME || s.row_step(*s.step, eb) % a.early_period != 0;
    }
    if (!a.kv_prefetch && !early) griddep_wait();
    char *ring = dsm;
    float *s_q = reinterpret_cast<float *>(dsm + (size_t)NW * NST * Gm::kPageBytes);
    float *cstate = s_q + (sizeof(T) == 4 ? G * D : 0);  // [G][D] acc, then m[16], l[16]
    float *cm = cstate + G * D, *cl = cm + 16;

    const int bh = blockIdx.x / S, rank = blockIdx.x % S;
    const HeadInfo hd = head_info(s, a, bh);
    const int n_att = hd.n_att;
    const int nwt = S * NW, kw = rank * NW + w;
    const int j0 = (int)((int64_t)n_att * kw / nwt);
    const int n_e = (int)((int64_t)n_att * (kw + 1) / nwt) - j0;
    const int b = bh / s.H, h = bh % s.H;
    const int64_t qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    const int last_fill = hd.n_tok - (hd.n_pages - 1) * kPageSize;  // tokens in the last page

    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    fence_mbar_init();
    __syncthreads();

    // entries are resolved 32 at a time (lane l owns entry 32c + l of chunk c)
    int cur_blk = 0, nxt_blk = 0;
    {
        const int j = j0 + lane;
        if (lane < n_e) cur_blk = resolve_block(s, hd, entry_page(s, hd, j));
        if (lane + 32 < n_e) nxt_blk = resolve_block(s, hd, entry_page(s, hd, j + 32));
    }
    const char *pool = reinterpret_cast<const char *>(s.pool);
    char *myring = ring + (size_t)w * NST * Gm::kPageBytes;
    uint64_t *mybars = bars + w * NST;
    int chunk = 0;  // chunk of cur_blk
#pragma unroll
    for (int i = 0; i < NST; ++i) {
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i);  // i < NST <= 32: chunk 0
        if (lane == 0 && i < n_e) {
            if (blk > 0) {
                mbar_arrive_expect_tx(&mybars[i], Gm::kPageBytes);
                bulk_page(myring + (size_t)i * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes,
                          Gm::kPageBytes, &mybars[i]);
            } else {
                mbar_arrive_expect_tx(&mybars[i], 0);
            }
        }
    }
    if constexpr (FC_L2_PREFETCH > 0) {
#pragma unroll
        for (int i = NST; i < NST + FC_L2_PREFETCH; ++i) {
            const int pblk = __shfl_sync(0xffffffffu, i < 32 ? cur_blk : nxt_blk, i & 31);
            if (lane == 0 && i < n_e && pblk > 0) bulk_prefetch_l2(pool + (int64_t)pblk * Gm::kPageBytes, Gm::kPageBytes);
        }
    }
    const unsigned long long t_issued = trace ? gtimer() : 0ull;

    if (a.kv_prefetch && !early) griddep_wait();  // q and the new token come from the previous launch
    if constexpr (sizeof(T) == 4) {
        const float *qg = reinterpret_cast<const float *>(a.q) + qoff;
        for (int i = tid; i < G * D; i += blockDim.x) s_q[i] = qg[i];
        __syncthreads();
    }
    typename std::conditional<sizeof(T) == 2, Bf16Attn<D>, F32Warp<D>>::type st;
    if constexpr (sizeof(T) == 4) st.init(s_q, G, lane);
    else st.init(reinterpret_cast<const T *>(a.q) + qoff, G, lane);
    // the warp holding the head's last entry loads the new token (and the
    // summary row it folds into) now, not when it reaches that page
    TokenPatch<T, D> tp;
    const int tok_slot = (hd.n_tok - 1) % kPageSize;
    // is the head's last attended entry its last (partial) page? (read now,
    // off the critical path of the last page)
    const bool last_is_last_page =
        n_e > 0 && j0 + n_e == n_att && entry_page(s, hd, n_att - 1) == hd.n_pages - 1;
    if (a.k_new != nullptr && n_e > 0 && j0 + n_e == n_att) {
        const int64_t nk = ((int64_t)b * s.H + h) * D;
        tp.load(s, reinterpret_cast<const T *>(a.k_new) + nk, reinterpret_cast<const T *>(a.v_new) + nk, hd.hx,
                hd.n_pages - 1, tok_slot, lane);
    }
    for (int i = 0; i < n_e; ++i) {
        // advance the resolution window when consumption enters a new chunk
        if (i > 0 && (i & 31) == 0) {
            cur_blk = nxt_blk;
            ++chunk;
            const int j = j0 + (chunk + 1) * 32 + lane;
            nxt_blk = (j < j0 + n_e) ? resolve_block(s, hd, entry_page(s, hd, j)) : 0;
        }
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i & 31);
        const int ni = i + NST;  // entry to issue after this one
        const int nb_cur = __shfl_sync(0xffffffffu, cur_blk, ni & 31);
        const int nb_nxt = __shfl_sync(0xffffffffu, nxt_blk, ni & 31);
        const int nblk = (ni >> 5) == chunk ? nb_cur : nb_nxt;
        const int stg = i % NST;
        mbar_wait(&mybars[stg], (i / NST) & 1);
        if (blk > 0) {
            char *stage = myring + (size_t)stg * Gm::kPageBytes;
            const bool last = (j0 + i == n_att - 1);
            const int page_is_last = last && last_is_last_page;
            if (last && a.k_new != nullptr)
                tp.apply(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk), tok_slot, hd.hx,
                         hd.n_pages - 1, lane);
#ifndef FC_SKIP_PAGE_MATH  // profiling knob: the page pipeline without the math
            st.page(stage, page_is_last ? last_fill : kPageSize, a.scale_log2, lane);
#endif
        }
        __syncwarp();
        if constexpr (FC_L2_PREFETCH > 0) {
            const int pi = ni + FC_L2_PREFETCH;  // within the current or next 32-entry chunk
            const int pb_cur = __shfl_sync(0xffffffffu, cur_blk, pi & 31);
            const int pb_nxt = __shfl_sync(0xffffffffu, nxt_blk, pi & 31);
            const int pblk = (pi >> 5) == chunk ? pb_cur : ((pi >> 5) == chunk + 1 ? pb_nxt : 0);
            if (lane == 0 && pi < n_e && pblk > 0)
                bulk_prefetch_l2(pool + (int64_t)pblk * Gm::kPageBytes, Gm::kPageBytes);
        }
        if (lane == 0 && ni < n_e) {
            if (FC_REFILL_FENCE) fence_proxy_async_smem();
            if (nblk > 0) {
                mbar_arrive_expect_tx(&mybars[stg], Gm::kPageBytes);
                bulk_page(myring + (size_t)stg * Gm::kPageBytes, pool + (int64_t)nblk * Gm::kPageBytes,
                          Gm::kPageBytes, &mybars[stg]);
            } else {
                mbar_arrive_expect_tx(&mybars[stg], 0);
            }
        }
    }
    const unsigned long long t_loop = trace ? gtimer() : 0ull;

    // ---- merge the warps of this CTA (ring is free once every warp is done)
    st.finalize();
    __syncthreads();
    float *scratch = reinterpret_cast<float *>(ring);  // [NW][G][D]
    for (int g = lane; g < 16; g += 32) { s_wm[w][g] = -INFINITY; s_wl[w][g] = 0.f; }
    __syncwarp();
    st.store_partial(scratch + (size_t)w * G * D, s_wm[w], s_wl[w], G, lane);
    __syncthreads();
    T *out = reinterpret_cast<T *>(a.out) + qoff;
    float *lse = a.lse ? a.lse + (int64_t)bh * G : nullptr;
    for (int e = tid; e < G * D; e += blockDim.x) {
        const int g = e / D;
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) M = fmaxf(M, s_wm[ww][g]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
            // idle warps hold m = -inf; a CTA whose warps are all idle (a cluster
            // rank with no attended pages) has M = -inf too: guard the -inf - -inf
            const float f = M == -INFINITY ? 0.f : exp2f(s_wm[ww][g] - M);
            L += s_wl[ww][g] * f;
            O += scratch[(size_t)ww * G * D + e] * f;
        }
        if (S == 1) {
            if (n_att > 0) {
                out[e] = T(O / L);
                if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
            }
        } else {
            cstate[e] = O;
            if (e % D == 0) { cm[g] = M; cl[g] = L; }
        }
    }
    if (S > 1) {  // ---- merge the cluster's CTAs into rank 0 through DSMEM
        namespace cg = cooperative_groups;
        cg::cluster_group cluster = cg::this_cluster();
        cluster.sync();
        if (rank == 0 && n_att > 0) {
            for (int e = tid; e < G * D; e += blockDim.x) {
                const int g = e / D;
                float M = -INFINITY;
                for (int r = 0; r < S; ++r) M = fmaxf(M, cluster.map_shared_rank(cm, r)[g]);
                float L = 0.f, O = 0.f;
                for (int r = 0; r < S; ++r) {
                    const float mr = cluster.map_shared_rank(cm, r)[g];
                    const float f = mr == -INFINITY ? 0.f : exp2f(mr - M);  // empty rank: 0, not NaN
                    L += cluster.map_shared_rank(cl, r)[g] * f;
                    O += cluster.map_shared_rank(cstate, r)[e] * f;
                }
                out[e] = T(O / L);
                if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
            }
        }
        cluster.sync();  // keep every rank's shared memory alive until rank 0 is done
    }
    // an early head still waits before exiting, so this launch completing
    // implies the scoring launch (and everything before it) completed
    if (early) griddep_wait();
    if (trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        unsigned long long *tw = trace + (size_t)blockIdx.x * 4;
        tw[0] = t_entry;
        tw[1] = t_issued;
        tw[2] = t_loop;
        tw[3] = gtimer() | 0ull;
        (void)smid;
    }
}

// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// Balanced variant for batches with fewer heads than CTA slots (e.g. 128
// heads on 148 SMs): the concatenation of every head's attended pages is cut
// into one equal range per CTA (all SMs busy), and each CTA's range into one
// contiguous sub-range per warp.  A warp keeps one softmax state per head it
// touches: a head that lies inside the warp is written directly; a head cut
// by the warp's start is parked in shared memory (slot A), one cut by its end
// stays in registers until the loop ends (slot B, in the freed ring).  The CTA
// then merges its slots per head: heads inside the CTA are written; the head
// continuing into the next CTA is published as a partial (slot = CTA index,
// release flag) BEFORE this CTA waits for anything; the head that started in
// earlier CTAs is finished by this CTA (its owner) after acquiring their
// partials.  All CTAs are co-resident (grid = SMs x occupancy), waits only go
// to lower CTA indices, so there is no deadlock; results are deterministic.
template <typename T, int D, int NST, int NW>
__global__ void __launch_bounds__(NW * 32)
attn_bal_kernel(StoreView s, AttnArgs a, int n_heads) {
    using Gm = AttnGeom<T, D>;
    // dynamic: ring [NW][NST][page] | slotA [NW][G][D] f32 | (fp32) q [NW][G][D] | prefix [n_heads+1]
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ float s_sm[2 * NW][16], s_sl[2 * NW][16];
    __shared__ int s_shead[2 * NW];
    __shared__ int s_wsum[NW];
    __shared__ int s_heads[4 * NW], s_nheads;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = s.G;
    unsigned long long *trace = g_attn_trace;
    const unsigned long long t_entry = trace ? gtimer() : 0ull;
    griddep_launch_dependents();
    if (!a.kv_prefetch) griddep_wait();
    char *ring = dsm;
    float *slotA = reinterpret_cast<float *>(dsm + (size_t)NW * NST * Gm::kPageBytes);
    float *s_q = slotA + (size_t)NW * G * D;
    int *prefix = reinterpret_cast<int *>(s_q + (sizeof(T) == 4 ? (size_t)NW * G * D : 0));
    float *slotB = reinterpret_cast<float *>(ring);  // reused once every warp is done

    // ---- prefix of attended pages over the heads of this layer
    {
        int carry = 0;
        for (int c0 = 0; c0 < n_heads; c0 += blockDim.x) {
            const int bh = c0 + tid;
            const int cnt = bh < n_heads ? head_info(s, a, bh).n_att : 0;
            int x = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) s_wsum[w] = x;
            __syncthreads();
            int before = carry, total = 0;
            for (int ww = 0; ww < NW; ++ww) {
                if (ww < w) before += s_wsum[ww];
                total += s_wsum[ww];
            }
            if (bh < n_heads) prefix[bh] = before + x - cnt;
            carry += total;
            __syncthreads();
        }
        if (tid == 0) prefix[n_heads] = carry;
    }
    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    if (tid < 2 * NW) s_shead[tid] = -1;
    fence_mbar_init();
    __syncthreads();
    const int total = prefix[n_heads];
    const int P = (total + gridDim.x - 1) / gridDim.x;
    const int lo = min(total, (int)blockIdx.x * P), hi = min(total, lo + P);
    const int wl = lo + (int)((int64_t)(hi - lo) * w / NW);
    const int n_e = lo + (int)((int64_t)(hi - lo) * (w + 1) / NW) - wl;
    auto head_of = [&](int pos) {  // last head with prefix <= pos
        int l0 = 0, h0 = n_heads - 1;
        while (l0 < h0) {
            const int mid = (l0 + h0 + 1) >> 1;
            if (prefix[mid] <= pos) l0 = mid; else h0 = mid - 1;
        }
        return l0;
    };
    auto resolve = [&](int pos, int &blk, int &bh) {
        bh = head_of(pos);
        const HeadInfo hd = head_info(s, a, bh);
        blk = resolve_block(s, hd, entry_page(s, hd, pos - prefix[bh]));
    };
    // ---- per-warp entry window (32 at a time) + ring prologue
    int cur_blk = 0, cur_bh = 0, nxt_blk = 0, nxt_bh = 0;
    if (lane < n_e) resolve(wl + lane, cur_blk, cur_bh);
    if (lane + 32 < n_e) resolve(wl + lane + 32, nxt_blk, nxt_bh);
    const char *pool = reinterpret_cast<const char *>(s.pool);
    char *myring = ring + (size_t)w * NST * Gm::kPageBytes;
    uint64_t *mybars = bars + w * NST;
#pragma unroll
    for (int i = 0; i < NST; ++i) {
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i);
        if (lane == 0 && i < n_e) {
            if (blk > 0) {
                mbar_arrive_expect_tx(&mybars[i], Gm::kPageBytes);
                bulk_page(myring + (size_t)i * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes,
                          Gm::kPageBytes, &mybars[i]);
            } else {
                mbar_arrive_expect_tx(&mybars[i], 0);
            }
        }
    }
    if (a.kv_prefetch) griddep_wait();  // q and the new token come from the previous launch
    const unsigned long long t_issued = trace ? gtimer() : 0ull;

    typename std::conditional<sizeof(T) == 2, Bf16Attn<D>, F32Warp<D>>::type st;
    T *out = reinterpret_cast<T *>(a.out);
    const T *qall = reinterpret_cast<const T *>(a.q);
    float *myq = s_q + (size_t)w * G * D;
    int cur = -1, seg_start = 0, chunk = 0;
    HeadInfo hd{};
    int64_t qoff = 0;
    auto close_segment = [&](int end_pos, bool last_of_warp) {
        // segment of head `cur` covering [seg_start, end_pos) of this warp
        st.finalize();
        const bool whole = seg_start == prefix[cur] && end_pos == prefix[cur + 1];
        if (whole) {
            st.template store_final<T>(out + qoff, a.lse ? a.lse + (int64_t)cur * G : nullptr, G, lane);
        } else if (!last_of_warp) {  // cut by the warp start: park in slot A
            for (int g = lane; g < 16; g += 32) { s_sm[w][g] = -INFINITY; s_sl[w][g] = 0.f; }
            __syncwarp();
            st.store_partial(slotA + (size_t)w * G * D, s_sm[w], s_sl[w], G, lane);
            if (lane == 0) s_shead[w] = cur;
        }
        return whole;
    };
    bool last_whole = true;
    for (int i = 0; i < n_e; ++i) {
        if (i > 0 && (i & 31) == 0) {
            cur_blk = nxt_blk;
            cur_bh = nxt_bh;
            ++chunk;
            const int j = (chunk + 1) * 32 + lane;
            nxt_blk = 0;
            if (j < n_e) resolve(wl + j, nxt_blk, nxt_bh);
        }
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i & 31);
        const int bh = __shfl_sync(0xffffffffu, cur_bh, i & 31);
        const int ni = i + NST;
        const int nb_cur = __shfl_sync(0xffffffffu, cur_blk, ni & 31);
        const int nb_nxt = __shfl_sync(0xffffffffu, nxt_blk, ni & 31);
        const int nblk = (ni >> 5) == chunk ? nb_cur : nb_nxt;
        if (bh != cur) {
            if (cur >= 0) close_segment(wl + i, false);
            cur = bh;
            seg_start = wl + i;
            hd = head_info(s, a, bh);
            const int b = bh / s.H, h = bh % s.H;
            qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
            if constexpr (sizeof(T) == 4) {
                __syncwarp();
                for (int k2 = lane; k2 < G * D; k2 += 32) myq[k2] = reinterpret_cast<const float *>(qall)[qoff + k2];
                __syncwarp();
                st.init(myq, G, lane);
            } else {
                st.init(qall + qoff, G, lane);
            }
        }
        const int stg = i % NST;
        mbar_wait(&mybars[stg], (i / NST) & 1);
        if (blk > 0) {
            char *stage = myring + (size_t)stg * Gm::kPageBytes;
            const int j = wl + i - prefix[bh];
            const bool last_entry = (j == hd.n_att - 1);
            const bool last_page = last_entry && entry_page(s, hd, j) == hd.n_pages - 1;
            if (last_page && a.k_new != nullptr) {
                const int b = bh / s.H, h = bh % s.H;
                const int64_t nk = ((int64_t)b * s.H + h) * D;
                patch_token<T, D>(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk),
                                  (hd.n_tok - 1) % kPageSize, hd.hx, hd.n_pages - 1,
                                  reinterpret_cast<const T *>(a.k_new) + nk,
                                  reinterpret_cast<const T *>(a.v_new) + nk, lane);
            }
            st.page(stage, last_page ? hd.n_tok - (hd.n_pages - 1) * kPageSize : kPageSize,
                    a.scale_log2, lane);
        }
        __syncwarp();
        if (lane == 0 && ni < n_e) {
            if (FC_REFILL_FENCE) fence_proxy_async_smem();
            if (nblk > 0) {
                mbar_arrive_expect_tx(&mybars[stg], Gm::kPageBytes);
                bulk_page(myring + (size_t)stg * Gm::kPageBytes, pool + (int64_t)nblk * Gm::kPageBytes,
                          Gm::kPageBytes, &mybars[stg]);
            } else {
                mbar_arrive_expect_tx(&mybars[stg], 0);
            }
        }
    }
    if (cur >= 0) last_whole = close_segment(wl + n_e, true);
    const unsigned long long t_loop = trace ? gtimer() : 0ull;
    __syncthreads();  // every warp done with its ring: slot B may use it
    if (cur >= 0 && !last_whole) {
        for (int g = lane; g < 16; g += 32) { s_sm[NW + w][g] = -INFINITY; s_sl[NW + w][g] = 0.f; }
        __syncwarp();
        st.store_partial(slotB + (size_t)w * G * D, s_sm[NW + w], s_sl[NW + w], G, lane);
        if (lane == 0) s_shead[NW + w] = cur;
    }
    __syncthreads();
    // ---- heads with parked states, ascending
    if (tid == 0) {
        int n = 0;
        for (int k2 = 0; k2 < 2 * NW; ++k2) {
            const int h2 = s_shead[k2];
            if (h2 < 0) continue;
            bool seen = false;
            for (int t2 = 0; t2 < n; ++t2) seen |= (s_heads[t2] == h2);
            if (!seen) s_heads[n++] = h2;
        }
        for (int x = 1; x < n; ++x)  // insertion sort (n <= 2*NW)
            for (int y = x; y > 0 && s_heads[y - 1] > s_heads[y]; --y) {
                const int t3 = s_heads[y]; s_heads[y] = s_heads[y - 1]; s_heads[y - 1] = t3;
            }
        s_nheads = n;
    }
    __syncthreads();
    const int nh = s_nheads;
    // continuing head first (publish before waiting), then the others
    for (int pass = 0; pass < 2; ++pass) {
        for (int t2 = 0; t2 < nh; ++t2) {
            const int h2 = s_heads[t2];
            const bool cont = prefix[h2 + 1] > hi;
            if (cont != (pass == 0)) continue;
            const bool owner_wait = !cont && prefix[h2] < lo;
            const int c_first = owner_wait ? prefix[h2] / P : 0;
            const int b = h2 / s.H, hh = h2 % s.H;
            T *o = out + ((int64_t)b * s.H * G + (int64_t)hh * G) * D;
            if (owner_wait) {  // acquire the partials of the earlier CTAs covering this head
                if (tid < (int)blockIdx.x - c_first) {
                    const int* f = a.counters + c_first + tid;
                    int v;
                    do {
                        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                    } while (v == 0);
                }
                __syncthreads();
            }
            for (int e = tid; e < G * D; e += blockDim.x) {
                const int g = e / D;
                float M = -INFINITY;
                for (int k2 = 0; k2 < 2 * NW; ++k2)
                    if (s_shead[k2] == h2) M = fmaxf(M, s_sm[k2][g]);
                if (owner_wait)
                    for (int c2 = c_first; c2 < (int)blockIdx.x; ++c2) M = fmaxf(M, __ldcg(a.part_m + c2 * 16 + g));
                float L = 0.f, O = 0.f;
                for (int k2 = 0; k2 < 2 * NW; ++k2) {
                    if (s_shead[k2] != h2) continue;
                    const float f = M == -INFINITY ? 0.f : exp2f(s_sm[k2][g] - M);
                    L += s_sl[k2][g] * f;
                    O += (k2 < NW ? slotA + (size_t)k2 * G * D : slotB + (size_t)(k2 - NW) * G * D)[e] * f;
                }
                if (owner_wait)
                    for (int c2 = c_first; c2 < (int)blockIdx.x; ++c2) {
                        const float f = M == -INFINITY ? 0.f : exp2f(__ldcg(a.part_m + c2 * 16 + g) - M);
                        L += __ldcg(a.part_l + c2 * 16 + g) * f;
                        O += __ldcg(a.part_o + ((int64_t)c2 * G * D) + e) * f;
                    }
                if (cont) {
                    a.part_o[(int64_t)blockIdx.x * G * D + e] = O;
                    if (e % D == 0) { a.part_m[blockIdx.x * 16 + g] = M; a.part_l[blockIdx.x * 16 + g] = L; }
                } else {
                    o[e] = T(O / L);
                    if (a.lse && e % D == 0) a.lse[(int64_t)h2 * G + g] = (M + log2f(L)) * 0.69314718055994531f;
                }
            }
            __syncthreads();
            if (cont && tid == 0) {  // publish: partial visible before the flag
                __threadfence();
                asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.counters + blockIdx.x), "r"(1) : "memory");
            }
            if (owner_wait && tid < (int)blockIdx.x - c_first) a.counters[c_first + tid] = 0;  // consumed
        }
    }
    if (trace && tid == 0) {
        unsigned long long *tw = trace + (size_t)blockIdx.x * 4;
        tw[0] = t_entry;
        tw[1] = t_issued;
        tw[2] = t_loop;
        tw[3] = gtimer();
    }
}

// CTA shapes: bf16 8 warps x 3 stages (192 KiB ring, one CTA per SM); fp32
// (correctness mode, 2x page bytes) 4 warps.
template <typename T, int D, int NST, int NW>
static size_t attn_smem(const StoreView &s) {
    using Gm = AttnGeom<T, D>;
    const size_t ring = (size_t)NW * NST * Gm::kPageBytes;
    const size_t merge = (size_t)NW * s.G * D * sizeof(float);  // scratch lives in the ring
    return (ring > merge ? ring : merge) + (size_t)(sizeof(T) == 4 ? s.G * D : 0) * sizeof(float) +
           ((size_t)s.G * D + 32) * sizeof(float);
}

template <typename T, int D, int NST, int NW>
static size_t attn_bal_smem(const StoreView &s, int n_heads) {
    using Gm = AttnGeom<T, D>;
    return (size_t)NW * NST * Gm::kPageBytes + (size_t)NW * s.G * D * sizeof(float) +
           (size_t)(sizeof(T) == 4 ? NW * s.G * D : 0) * sizeof(float) + (size_t)(n_heads + 1) * sizeof(int);
}

template <typename T, int D, int NST, int NW>
static int attn_bal_ctas_per_sm_t(const StoreView &s, int n_heads) {
    const size_t smem = attn_bal_smem<T, D, NST, NW>(s, n_heads);
    auto kern = attn_bal_kernel<T, D, NST, NW>;
    int occ = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();  // does not fit: not an error of the caller's stream
        return 0;
    }
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem);
    return occ;
}

template <typename T, int D, int NST, int NW>
static int attn_ctas_per_sm_t(const StoreView &s) {
    const size_t smem = attn_smem<T, D, NST, NW>(s);
    auto kern = attn_kernel<T, D, NST, NW>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 1;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, smem);
    return occ < 1 ? 1 : occ;
}

#ifndef FC_ATTN_NW
#define FC_ATTN_NW 8    // bf16 warps per CTA
#endif
#ifndef FC_ATTN_NST
#define FC_ATTN_NST 3   // bf16 d=128 ring stages per warp (NW * NST * 8 KiB <= ~200 KiB)
#endif
#define FC_ATTN_DISPATCH(dtype, D, CALL)                                            \
    ((dtype) == FC_BF16 ? ((D) == 128 ? CALL(__nv_bfloat16, 128, FC_ATTN_NST, FC_ATTN_NW)                \
                                      : CALL(__nv_bfloat16, 64, 2 * FC_ATTN_NST, FC_ATTN_NW))            \
                        : ((D) == 128 ? CALL(float, 128, 3, 4) : CALL(float, 64, 6, 4)))

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

// CTAs per head (cluster size): the largest power of two <= 16 that keeps
// heads * S within one wave and gives every warp at least two pages.
// Variant choice: 0 = cluster-per-head kernel always (default: measured faster
// than the balanced variant at 32-128 heads and equal within noise at 8-16);
// 1 = balanced all-SM variant whenever heads <= half the CTA slots; -1 = that
// rule too (kept for the test hook).
#ifndef FC_ATTN_MODE_DEFAULT
#define FC_ATTN_MODE_DEFAULT 0
#endif
static int g_attn_mode = FC_ATTN_MODE_DEFAULT;
void set_attn_mode(int m) { g_attn_mode = m; }

#ifndef FC_ATTN_SMAX
#define FC_ATTN_SMAX kMaxClusterCtas  // largest automatic cluster size
#endif
int attn_split(const StoreView &s, int dtype, int batch, int max_pages, int n_ctas) {
    const int n_heads = batch * s.H;
#define FC_OCC(T, DD, N, W) attn_ctas_per_sm_t<T, DD, N, W>(s)
    const int occ = FC_ATTN_DISPATCH(dtype, s.D, FC_OCC);  // (also sets the kernel's smem attribute)
#undef FC_OCC
    if (n_ctas > 0) return n_ctas;  // explicit split (profiling, tests)
    const int64_t slots = (int64_t)occ * num_sms();
    if (g_attn_mode != 0 && (int64_t)n_heads * 2 <= slots) {  // far fewer heads than CTA slots: balanced all-SM variant
#define FC_BOCC(T, DD, N, W) attn_bal_ctas_per_sm_t<T, DD, N, W>(s, n_heads)
        const int bocc = FC_ATTN_DISPATCH(dtype, s.D, FC_BOCC);
#undef FC_BOCC
        if (bocc >= 1) return -(bocc * num_sms());
    }
    int S = 1;
    while (2 * S <= FC_ATTN_SMAX && 2 * S <= max_cluster() && (int64_t)n_heads * 2 * S <= slots &&
           2 * S * 4 * 2 <= max_pages)
        S *= 2;
    return S;
}

#ifndef FC_ATTN_CLUSTER1
#define FC_ATTN_CLUSTER1 0
#endif
template <typename T, int D, int NST, int NW>
static cudaError_t launch_attn_t(const StoreView &s, const AttnArgs &a, int batch, cudaStream_t st) {
    const int n_heads = batch * s.H;
    if (a.max_splits < 0) {  // balanced variant on -max_splits CTAs
        return launch_pdl(attn_bal_kernel<T, D, NST, NW>, dim3(-a.max_splits), dim3(NW * 32),
                          attn_bal_smem<T, D, NST, NW>(s, n_heads), st, s, a, n_heads);
    }
    const int S = a.max_splits;
    const size_t smem = attn_smem<T, D, NST, NW>(s);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n_heads * S);
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = S;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (S > 1 || FC_ATTN_CLUSTER1) ? 2 : 1;  // S = 1: a plain launch
    return cudaLaunchKernelEx(&cfg, attn_kernel<T, D, NST, NW>, s, a, S);
}

cudaError_t set_attn_trace(void *p) {
    return cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p));
}

cudaError_t launch_attn(const StoreView &s, int dtype, const AttnArgs &a, int batch, cudaStream_t st) {
    if (a.max_splits == 0 || a.max_splits > kMaxClusterCtas ||
        (int64_t)batch * s.H * (a.max_splits > 0 ? a.max_splits : 1) > 2147483647ll)
        return cudaErrorInvalidValue;
#define FC_LAUNCH(T, DD, N, W) launch_attn_t<T, DD, N, W>(s, a, batch, st)
    return FC_ATTN_DISPATCH(dtype, s.D, FC_LAUNCH);
#undef FC_LAUNCH
}

// workspace: balanced variant (split < 0): per-CTA flags + partials; else a
// small scratch (the cluster variant merges in DSMEM)
size_t attn_workspace_bytes(const StoreView &s, int, int split) {
    if (split >= 0) return 256;
    const size_t n = (size_t)(-split);
    return ((n * sizeof(int32_t) + 255) & ~(size_t)255) + n * 32 * sizeof(float) + n * s.G * s.D * sizeof(float);
}

}  // namespace fc
