// attn_run.cu — subsystem (3), persistent form: GQA paged sparse decode
// attention for a RUN of consecutive layers in one launch, every SM busy.
//
// Reference semantics are those of sparse_decode (attention.py:85-111) per
// (layer, head), exactly as attn_kernel (sparse_decode.cu): softmax(q·Kᵀ/√d)·V
// over the attended pages in ascending page order, residency violations
// flagged (attention.py:101-105), the decode append fused in
// (update_minmax, scoring.py:59-69).
//
// Why a second kernel: at config 2 one head per CTA leaves 20 of 148 SMs idle,
// and every per-layer launch pays a dependent-load prologue (selection ->
// table -> first copy) and a tail where SMs that share a TPC with an idle SM
// run faster than the rest.  Here the grid is one CTA per SM for the whole
// run of layers and the WARP is the unit of work:
//
//  * plan: per layer, the attended pages of all heads are concatenated (head
//    order) and cut into one equal contiguous range per warp of the grid
//    (1184 warps at 148 SMs x 8).  Each warp computes its own plan — head
//    prefix sums into shared memory, then the physical block of every entry
//    of its range — one layer AHEAD of consumption;
//  * stream: each warp owns a ring of NST page stages (cp.async.bulk of the
//    whole 8 KiB page onto an mbarrier, as attn_kernel).  The issue pointer
//    runs NST entries ahead of consumption ACROSS the layer boundary, so the
//    pages of layer l+1 are in flight while layer l finishes;
//  * layer dependency: a layer's q (and its new token) may be consumed only
//    after every output of the previous layer is written — a grid barrier
//    (release/acquire counter) between layers models the decoder's layer
//    chain.  Page copies do not depend on it and keep HBM busy through it;
//  * merge: a head cut across warps publishes per-warp partials (unnormalised
//    acc, running max, sum) to L2; the warp that arrives last on the head's
//    counter merges all of them in ascending range order (deterministic) and
//    writes the output.  No CTA-wide synchronisation anywhere: warps are
//    independent except for the layer barrier.
//
// Co-residency: the grid is <= SMs x occupancy(1), so every CTA is resident
// once the previous kernel drains; dependents are released (PDL) only after
// the first in-kernel barrier proved all CTAs resident.
#include "attn_warp.cuh"

namespace fc {

// Optional per-warp timeline (globaltimer ns) for profiling: [warps][33][8];
// [li] = loop top, next layer planned, barrier passed, layer consumed,
// ns in segment closes, ns in merges, segments, merges;
// [32] = entry, first plan done, exit.  Null in production.
__device__ unsigned long long *g_run_trace = nullptr;

FC_DEVINL unsigned long long run_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int kRunMaxHeadChunks = 8;   // heads per layer <= 256
constexpr int kRunMaxHeads = 32 * kRunMaxHeadChunks;

FC_DEVINL void red_release_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FC_DEVINL uint32_t ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// CTA-scope flag in shared memory: atomic read / write with block fences
// (acquire / release semantics; atomics also keep racecheck informed)
FC_DEVINL int ld_acquire_cta(int *p) {
    const int v = atomicAdd(p, 0);
    __threadfence_block();
    return v;
}
FC_DEVINL void st_release_cta(int *p, int v) {
    __threadfence_block();
    atomicExch(p, v);
}

// per-warp plan of one layer: [prefix: nh+1 ints][blk: maxr][bh: maxr][pg: maxr]
struct RunPlan {
    int *prefix, *blk, *bh, *pg;
    __host__ __device__ static size_t ints(int nh, int maxr) { return (size_t)((nh + 1 + 3) & ~3) + 3 * (size_t)((maxr + 3) & ~3); }
    FC_DEVINL void bind(int *base, int nh, int maxr) {
        prefix = base;
        blk = base + ((nh + 1 + 3) & ~3);
        bh = blk + ((maxr + 3) & ~3);
        pg = bh + ((maxr + 3) & ~3);
    }
};

// warp owning position p of a layer cut into weff equal ranges of t entries
FC_DEVINL int run_warp_of(int64_t p, int weff, int64_t t) {
    return (int)(((p + 1) * weff + t - 1) / t) - 1;
}
FC_DEVINL int run_range_start(int w, int weff, int64_t t) { return (int)(t * w / weff); }

struct RunLayer {
    int n, ws, T, weff;
};

// Plan layer l for warp gw: prefix over heads, this warp's range, and the
// physical block / head / page of every entry in it.  Warp-collective.
// Dependent global round trips: seq_len + n_sel (+ the last selected page
// when attend_appended), then sel[j], then the table.  Per-head values reach
// the entry lanes by shuffles (lane bh % 32 of chunk bh / 32 holds them).
FC_DEVINL RunLayer run_plan(const StoreView &s, const RunArgs &a, int l, int nh, RunPlan &pl, int gw,
                            int W, int lane) {
    int ntok[kRunMaxHeadChunks], nsel[kRunMaxHeadChunks], hi[kRunMaxHeadChunks], cnt[kRunMaxHeadChunks];
#pragma unroll
    for (int k = 0; k < kRunMaxHeadChunks; ++k) {  // loads of every chunk in flight together
        const int bh = k * 32 + lane;
        ntok[k] = 0; nsel[k] = 0;
        if (bh < nh) {
            const int b = bh / s.H, h = bh % s.H;
            ntok[k] = s.decodes(b) ? s.seq_len[b] + a.extra_tokens : 0;
            nsel[k] = s.n_sel[s.hix(b, l, h)];
        }
    }
#pragma unroll
    for (int k = 0; k < kRunMaxHeadChunks; ++k) {
        const int bh = k * 32 + lane;
        hi[k] = -1;
        if (a.attend_appended && bh < nh && nsel[k] > 0) {
            const int b = bh / s.H, h = bh % s.H;
            hi[k] = s.sel[(int64_t)s.hix(b, l, h) * s.SELCAP + nsel[k] - 1];
        }
    }
#pragma unroll
    for (int k = 0; k < kRunMaxHeadChunks; ++k) {
        cnt[k] = 0;
        if (k * 32 + lane < nh && ntok[k] > 0) {
            const int n_pages = (ntok[k] + kPageSize - 1) / kPageSize;
            cnt[k] = a.attend_appended ? nsel[k] + max(0, n_pages - 1 - hi[k]) : nsel[k];
        }
    }
    int carry = 0, maxa = 0;
#pragma unroll
    for (int k = 0; k < kRunMaxHeadChunks; ++k) {
        if (k * 32 >= nh) break;
        maxa = max(maxa, cnt[k]);
        int x = cnt[k];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (k * 32 + lane < nh) pl.prefix[k * 32 + lane] = carry + x - cnt[k];
        carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) pl.prefix[nh] = carry;
    __syncwarp();
    RunLayer r;
    r.T = carry;
    maxa = __reduce_max_sync(0xffffffffu, maxa);
    // equal ranges of >= min_pages entries, and at most 31 parts per head
    // (run_merge merges <= 32): ranges of >= ceil(maxa / 30) entries
    r.weff = min(W, max(1, min(carry / a.min_pages, carry / max(1, (maxa + 29) / 30))));
    r.ws = 0;
    r.n = 0;
    if (gw < r.weff && carry > 0) {
        r.ws = run_range_start(gw, r.weff, carry);
        r.n = run_range_start(gw + 1, r.weff, carry) - r.ws;
    }
    if (r.n > a.maxr) {  // host sizing guarantees this never happens
        if (lane == 0) set_error(s.err, FC_ERR_RUN_RANGE);
        r.n = a.maxr;
    }
    for (int i0 = 0; i0 < r.n; i0 += 32) {
        const int i = i0 + lane;
        int bh = 0;
        if (i < r.n) {
            const int p = r.ws + i;
            int lo = 0, up = nh - 1;  // last head with prefix <= p
            while (lo < up) {
                const int mid = (lo + up + 1) >> 1;
                if (pl.prefix[mid] <= p) lo = mid; else up = mid - 1;
            }
            bh = lo;
        }
        int my_ntok = 0, my_nsel = 0, my_hi = -1;
#pragma unroll
        for (int k = 0; k < kRunMaxHeadChunks; ++k) {
            if (k * 32 >= nh) break;
            const int t0 = __shfl_sync(0xffffffffu, ntok[k], bh & 31);
            const int t1 = __shfl_sync(0xffffffffu, nsel[k], bh & 31);
            const int t2 = __shfl_sync(0xffffffffu, hi[k], bh & 31);
            if ((bh >> 5) == k) { my_ntok = t0; my_nsel = t1; my_hi = t2; }
        }
        if (i < r.n) {
            const int b = bh / s.H, h = bh % s.H;
            const int hx = s.hix(b, l, h);
            const int j = r.ws + i - pl.prefix[bh];
            const int n_pages = (my_ntok + kPageSize - 1) / kPageSize;
            const int page = j < my_nsel ? s.sel[(int64_t)hx * s.SELCAP + j] : my_hi + 1 + (j - my_nsel);
            int blk = 0;
            if (page >= 0 && page < n_pages) blk = s.table[s.table_off(hx, page)];
            if (blk == FC_NULL_BLOCK) {  // residency violation (attention.py:101-105)
                set_error(s.err, FC_ERR_NULL_READ);
                blk = -1;
            }
            pl.blk[i] = blk;
            pl.bh[i] = bh;
            const int n_att = pl.prefix[bh + 1] - pl.prefix[bh];
            const bool last_page = (j == n_att - 1) && page == n_pages - 1;
            const int fill = my_ntok - (n_pages - 1) * kPageSize;  // 1..16
            pl.pg[i] = page | (last_page ? (int)(0x80000000u | ((uint32_t)fill << 24)) : 0);
        }
    }
    __syncwarp();
    return r;
}

// Merge the np (<= 32) partials of one head, parts wa..wa+np-1 in range
// order: lane x stages part x's running maxima in shared memory (fs[32][16])
// and keeps its sums in registers; row maxima / sums are warp reductions and
// fs is overwritten with the per-(part, row) factors; then every lane
// accumulates its float4 columns over all parts (4 chunks x 4 parts of loads
// in flight).  Writes out [G][D] and lse [G].
template <typename T, int D>
FC_DEVINL void run_merge(const float *part, int pstride, int G, int wa, int np, int h0, int weff, int64_t tt,
                         T *out, float *lse, float *fs, int lane) {
    int base = 0;
    float lr[16];
    if (lane < np) {
        const int x = wa + lane;
        base = (x * 2 + (run_range_start(x, weff, tt) >= h0 ? 0 : 1)) * pstride;
    }
    float mr[16];
#pragma unroll
    for (int g = 0; g < 16; ++g) {  // every load issued before the first use
        lr[g] = 0.f;
        mr[g] = -INFINITY;
        if (g < G && lane < np) {
            mr[g] = __ldcg(part + base + G * D + g);
            lr[g] = __ldcg(part + base + G * D + 16 + g);
        }
    }
    float Lrow = 1.f, Mrow = 0.f;  // lane g < G keeps row g
#pragma unroll
    for (int g = 0; g < 16; ++g) {
        if (g < G) {
            const float mg = mr[g];
            const float M = warp_max(mg);
            const float f = (lane < np && M != -INFINITY) ? exp2f(mg - M) : 0.f;
            const float L = warp_sum(lr[g] * f);
            if (lane < np) fs[lane * 16 + g] = f;
            if (lane == g) { Lrow = L; Mrow = M; }
        }
    }
    __syncwarp();
    const int nitems = G * D / 4;
    for (int k0 = 0; k0 * 32 < nitems; k0 += 4) {
        float4 o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int x = 0; x < np; ++x) {
            const int bx = __shfl_sync(0xffffffffu, base, x);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int item = lane + 32 * (k0 + k);
                if (item < nitems) {
                    const float fx = fs[x * 16 + item * 4 / D];
                    const float4 v = __ldcg(reinterpret_cast<const float4 *>(part + bx) + item);
                    o[k].x += v.x * fx; o[k].y += v.y * fx; o[k].z += v.z * fx; o[k].w += v.w * fx;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int item = lane + 32 * (k0 + k);
            const int g = item * 4 / D;
            const float L = __shfl_sync(0xffffffffu, Lrow, g & 31);
            if (item < nitems) {
                const float inv = 1.f / L;
                T *dst = out + item * 4;
                dst[0] = T(o[k].x * inv); dst[1] = T(o[k].y * inv); dst[2] = T(o[k].z * inv); dst[3] = T(o[k].w * inv);
            }
        }
    }
    if (lse && lane < G) lse[lane] = (Mrow + log2f(Lrow)) * 0.69314718055994531f;
    __syncwarp();
}

template <typename T, int D, int NST, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
attn_run_kernel(StoreView s, RunArgs a) {
    using Gm = AttnGeom<T, D>;
    // dynamic: ring [NW][NST][page] | plans [NW][2] | (fp32) q [NW][G][D] | merge factors [NW][32][16]
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ int s_arrived, s_poller, s_pass;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = s.G;
    const int nh = a.batch * s.H;
    const int W = gridDim.x * NW, gw = blockIdx.x * NW + w;
    const size_t plan_ints = RunPlan::ints(nh, a.maxr);
    char *myring = dsm + (size_t)w * NST * Gm::kPageBytes;
    int *plan_base = reinterpret_cast<int *>(dsm + (size_t)NW * NST * Gm::kPageBytes) + (size_t)w * 2 * plan_ints;
    float *myq = reinterpret_cast<float *>(reinterpret_cast<int *>(dsm + (size_t)NW * NST * Gm::kPageBytes) +
                                           (size_t)NW * 2 * plan_ints) + (size_t)w * G * D;
    float *myfs = reinterpret_cast<float *>(reinterpret_cast<int *>(dsm + (size_t)NW * NST * Gm::kPageBytes) +
                                            (size_t)NW * 2 * plan_ints) +
                  (sizeof(T) == 4 ? (size_t)NW * G * D : 0) + (size_t)w * 32 * 16;
    uint64_t *mybars = bars + w * NST;
    const char *pool = reinterpret_cast<const char *>(s.pool);
    const int pstride = G * D + 32;  // partial: acc [G][D] | m [16] | l [16]

    if (lane < NST) mbar_init(&mybars[lane], 1);
    if (tid == 0) { s_arrived = 0; s_poller = 0; s_pass = 0; }
    fence_mbar_init();
    __syncthreads();  // the only CTA-wide barrier: shared state initialised
    if (a.nl == 1) griddep_launch_dependents();
    if (a.first_dep) griddep_wait();

    unsigned long long *trace = g_run_trace ? g_run_trace + (size_t)gw * 33 * 8 : nullptr;
    if (trace && lane == 0) trace[32 * 8 + 0] = run_gtimer();
    RunPlan pl[2];
    pl[0].bind(plan_base, nh, a.maxr);
    pl[1].bind(plan_base + plan_ints, nh, a.maxr);

    // issue pointer: (ili, ie) over the concatenation of planned layers
    int issued = 0, cons = 0;
    int ili = 0, ie = 0;
    RunLayer cur_l = run_plan(s, a, a.l0, nh, pl[0], gw, W, lane);
    RunLayer nxt_l{0, 0, 0, 1};
    bool nxt_ready = false;
    auto pump = [&](int li) {
        while (issued - cons < NST) {
            if (ili == li && ie >= cur_l.n) {
                if (!nxt_ready) break;
                ili = li + 1;
                ie = 0;
            }
            if (ili == li + 1 && ie >= nxt_l.n) break;
            const int blk = ((ili & 1) ? pl[1].blk : pl[0].blk)[ie];
            const int stg = issued % NST;
            if (lane == 0) {
                fence_proxy_async_smem();
                if (blk > 0) {
                    mbar_arrive_expect_tx(&mybars[stg], Gm::kPageBytes);
                    bulk_g2s(myring + (size_t)stg * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes,
                             Gm::kPageBytes, &mybars[stg]);
                } else {
                    mbar_arrive_expect_tx(&mybars[stg], 0);
                }
            }
            ++issued;
            ++ie;
        }
    };
    pump(0);
    if (trace && lane == 0) trace[32 * 8 + 1] = run_gtimer();

    typename std::conditional<sizeof(T) == 2, Bf16Attn<D>, F32Warp<D>>::type st;
    for (int li = 0; li < a.nl; ++li) {
        const int l = a.l0 + li;
        const RunPlan P = (li & 1) ? pl[1] : pl[0];
        const bool tr = trace && lane == 0 && li < 32;
        if (tr) trace[li * 8 + 0] = run_gtimer();
        // plan the next layer before waiting (its pages stream while we wait)
        if (li + 1 < a.nl) {
            nxt_l = run_plan(s, a, l + 1, nh, (li & 1) ? pl[0] : pl[1], gw, W, lane);
            nxt_ready = true;
            pump(li);
        }
        if (tr) trace[li * 8 + 1] = run_gtimer();
        if (li == 0 && !a.first_dep) griddep_wait();  // q and the new tokens come from the previous launch
        if (li > 0) {  // layer barrier: every output of layer l-1 is written
            // one elected warp per CTA polls the grid counter (CTA arrivals);
            // the others wait on the CTA's shared flag
            if (lane == 0) {
                while (ld_acquire_cta(&s_pass) < li) {
                    if (atomicCAS(&s_poller, li - 1, li) == li - 1) {
                        const uint32_t target = (uint32_t)li * gridDim.x;
                        while (ld_acquire(a.bar + 2 * a.l0) < target) __nanosleep(200);
                        st_release_cta(&s_pass, li);
                    } else {
                        __nanosleep(64);
                    }
                }
            }
            __syncwarp();
            if (li == 1) griddep_launch_dependents();  // every CTA is resident
        }
        if (tr) trace[li * 8 + 2] = run_gtimer();
        const T *q_l = reinterpret_cast<const T *>(a.q) + (int64_t)li * a.q_ls;
        const T *k_l = a.k_new ? reinterpret_cast<const T *>(a.k_new) + (int64_t)li * a.kv_ls : nullptr;
        const T *v_l = a.v_new ? reinterpret_cast<const T *>(a.v_new) + (int64_t)li * a.kv_ls : nullptr;
        T *out_l = reinterpret_cast<T *>(a.out) + (int64_t)li * a.o_ls;
        float *lse_l = a.lse ? a.lse + (int64_t)li * a.lse_ls : nullptr;

        int cur = -1, seg_start = 0;
        bool first_seg = true;
        unsigned long long tc_close = 0, tc_merge = 0;
        int n_seg = 0, n_merge = 0;
        auto close_segment = [&](int end_pos) {
            const unsigned long long tc0 = tr ? run_gtimer() : 0ull;
            ++n_seg;
            st.finalize();
            const int64_t qoff = (int64_t)cur * G * D;
            const int h0 = P.prefix[cur], h1 = P.prefix[cur + 1];
            if (seg_start == h0 && end_pos == h1) {
                st.template store_final<T>(out_l + qoff, lse_l ? lse_l + (int64_t)cur * G : nullptr, G, lane);
                if (tr) tc_close += run_gtimer() - tc0;
                return;
            }
            const int slot = first_seg ? 0 : 1;
            float *pp = a.part + ((int64_t)gw * 2 + slot) * pstride;
            st.store_partial(pp, pp + G * D, pp + G * D + 16, G, lane);
            __threadfence();
            __syncwarp();
            int old = 0;
            if (lane == 0) old = atomicAdd(a.head_cnt + cur, 1);
            old = __shfl_sync(0xffffffffu, old, 0);
            const int wa = run_warp_of(h0, cur_l.weff, cur_l.T), wb = run_warp_of(h1 - 1, cur_l.weff, cur_l.T);
            if (old != wb - wa) {
                if (tr) tc_close += run_gtimer() - tc0;
                return;
            }
            // last arriver: merge the parts of this head in range order
            const unsigned long long tm0 = tr ? run_gtimer() : 0ull;
            ++n_merge;
            __threadfence();
            run_merge<T, D>(a.part, pstride, G, wa, wb - wa + 1, h0, cur_l.weff, cur_l.T, out_l + qoff,
                            lse_l ? lse_l + (int64_t)cur * G : nullptr, myfs, lane);
            if (lane == 0) a.head_cnt[cur] = 0;  // every part arrived: reusable for the next layer
            if (tr) {
                const unsigned long long t9 = run_gtimer();
                tc_merge += t9 - tm0;
                tc_close += t9 - tc0;
            }
        };

        for (int e = 0; e < cur_l.n; ++e) {
            const int blk = P.blk[e], bh = P.bh[e], pg = P.pg[e];
            if (bh != cur) {
                if (cur >= 0) {
                    close_segment(cur_l.ws + e);
                    first_seg = false;
                }
                cur = bh;
                seg_start = cur_l.ws + e;
                const int64_t qoff = (int64_t)bh * G * D;
                if constexpr (sizeof(T) == 4) {
                    __syncwarp();
                    for (int k2 = lane; k2 < G * D; k2 += 32) myq[k2] = reinterpret_cast<const float *>(q_l)[qoff + k2];
                    __syncwarp();
                    st.init(myq, G, lane);
                } else {
                    st.init(q_l + qoff, G, lane);
                }
            }
            const int stg = cons % NST;
            mbar_wait(&mybars[stg], (cons / NST) & 1);
            if (blk > 0) {
                char *stage = myring + (size_t)stg * Gm::kPageBytes;
                const bool last_page = pg < 0;
                const int page = pg & 0x00ffffff, fill = (pg >> 24) & 0x1f;
                if (last_page && k_l != nullptr) {
                    const int b = bh / s.H, h = bh % s.H;
                    patch_token<T, D>(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk), fill - 1,
                                      s.hix(b, l, h), page, k_l + (int64_t)bh * D, v_l + (int64_t)bh * D, lane);
                }
                st.page(stage, last_page ? fill : kPageSize, a.scale_log2, lane);
            }
            __syncwarp();
            ++cons;
            pump(li);
        }
        if (cur >= 0) close_segment(cur_l.ws + cur_l.n);
        if (tr) {
            trace[li * 8 + 3] = run_gtimer();
            trace[li * 8 + 4] = tc_close;
            trace[li * 8 + 5] = tc_merge;
            trace[li * 8 + 6] = n_seg;
            trace[li * 8 + 7] = n_merge;
        }
        if (li + 1 < a.nl) {
            __threadfence();
            __syncwarp();
            if (lane == 0) {  // arrive; the CTA's last warp arrives on the grid counter
                const int before = atomicAdd(&s_arrived, 1);
                if (before == NW * (li + 1) - 1) {
                    __threadfence();
                    red_release_add(a.bar + 2 * a.l0, 1u);
                }
            }
            cur_l = nxt_l;
            nxt_ready = false;
            // the issue pointer may already be in layer li+1
            if (ili == li) { ili = li + 1; ie = 0; }
            pump(li + 1);
        }
    }
    if (trace && lane == 0) trace[32 * 8 + 2] = run_gtimer();
    if (a.nl > 1 && lane == 0) {  // the last warp out resets the barrier for the next launch
        __threadfence();
        const uint32_t old = atomicAdd(a.bar + 2 * a.l0 + 1, 1u);
        if (old == (uint32_t)W - 1) {
            a.bar[2 * a.l0] = 0u;
            a.bar[2 * a.l0 + 1] = 0u;
        }
    }
}

// ---------------------------------------------------------------------------
// host side

#ifndef FC_RUN_NW
#define FC_RUN_NW 8
#endif
#ifndef FC_RUN_NST
#define FC_RUN_NST 3
#endif
#ifndef FC_RUN_MIN_PAGES
#define FC_RUN_MIN_PAGES 4
#endif

#define FC_RUN_DISPATCH(dtype, D, CALL)                                                                  \
    ((dtype) == FC_BF16 ? ((D) == 128 ? CALL(__nv_bfloat16, 128, FC_RUN_NST, FC_RUN_NW)                    \
                                      : CALL(__nv_bfloat16, 64, 2 * FC_RUN_NST, FC_RUN_NW))                \
                        : ((D) == 128 ? CALL(float, 128, 3, 4) : CALL(float, 64, 6, 4)))

static int run_num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

template <typename T, int D, int NST, int NW>
static size_t run_smem(const StoreView &s, int nh, int maxr) {
    using Gm = AttnGeom<T, D>;
    return (size_t)NW * NST * Gm::kPageBytes + (size_t)NW * 2 * RunPlan::ints(nh, maxr) * sizeof(int) +
           (sizeof(T) == 4 ? (size_t)NW * s.G * D * sizeof(float) : 0) + (size_t)NW * 32 * 16 * sizeof(float);
}

template <typename T, int D, int NST, int NW>
static int run_warps_per_cta() { return NW; }

// entries per warp range: <= max(ceil(T / W), 2 * min_pages) (run_plan's cut)
static int run_maxr(int nh, int max_pages, int W) {
    const int64_t t = (int64_t)nh * max_pages;
    const int64_t per = (t + W - 1) / W;
    return (int)std::max<int64_t>(per, 2 * FC_RUN_MIN_PAGES) + 1;
}

template <typename T, int D, int NST, int NW>
static int run_plan_t(const StoreView &s, int batch, int max_pages, int *grid, int *maxr, size_t *smem) {
    const int nh = batch * s.H;
    if (nh < 1 || nh > kRunMaxHeads) return 0;
    const int g = run_num_sms();
    const int m = run_maxr(nh, max_pages, g * NW);
    const size_t sm = run_smem<T, D, NST, NW>(s, nh, m);
    auto kern = attn_run_kernel<T, D, NST, NW>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, sm) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        return 0;
    }
    if (grid) *grid = g;  // one CTA per SM: all co-resident
    if (maxr) *maxr = m;
    if (smem) *smem = sm;
    return 1;
}

// 0: per-head cluster persistent kernel when it fits (attn_persist.cu), else
// the warp-balanced one; 1: warp-balanced always (test / profiling hook)
static int g_run_mode = 0;
void set_run_mode(int m) { g_run_mode = m; }

int attn_run_supported(const StoreView &s, int dtype, int batch, int max_pages) {
    if (g_run_mode == 0 && attn_persist_split(s, dtype, batch, max_pages) > 0) return 1;
    if (dtype == FC_BF16 && s.G > 16) return 0;
    if (dtype == FC_F32 && s.G > 8) return 0;
#define FC_RP(T, DD, N, W_) run_plan_t<T, DD, N, W_>(s, batch, max_pages, nullptr, nullptr, nullptr)
    return FC_RUN_DISPATCH(dtype, s.D, FC_RP);
#undef FC_RP
}

// workspace: [L][2] u32 barrier counters | [256 heads] i32 head counters | partials
size_t attn_run_workspace_bytes(const StoreView &s, int dtype, int batch, int max_pages) {
    (void)batch; (void)max_pages;
    const int nw = (dtype == FC_BF16 ? FC_RUN_NW : 4) * run_num_sms();
    const size_t ctr = (((size_t)s.L * 2 * sizeof(uint32_t) + 255) & ~(size_t)255) + kRunMaxHeads * sizeof(int32_t);
    return ctr + (size_t)nw * 2 * (s.G * s.D + 32) * sizeof(float);
}

template <typename T, int D, int NST, int NW>
static cudaError_t launch_run_t(const StoreView &s, RunArgs a, int max_pages, cudaStream_t st) {
    int grid = 0, maxr = 0;
    size_t smem = 0;
    if (!run_plan_t<T, D, NST, NW>(s, a.batch, max_pages, &grid, &maxr, &smem)) return cudaErrorInvalidConfiguration;
    a.maxr = maxr;
    a.min_pages = FC_RUN_MIN_PAGES;
    return launch_pdl(attn_run_kernel<T, D, NST, NW>, dim3(grid), dim3(NW * 32), smem, st, s, a);
}

cudaError_t set_run_trace(void *p) { return cudaMemcpyToSymbol(g_run_trace, &p, sizeof(p)); }

cudaError_t launch_attn_run(const StoreView &s, int dtype, const RunArgs &a, int max_pages, void *ws,
                            cudaStream_t st) {
    RunArgs r = a;
    char *w = (char *)ws;
    r.bar = (uint32_t *)w;
    r.head_cnt = (int32_t *)(w + (((size_t)s.L * 2 * sizeof(uint32_t) + 255) & ~(size_t)255));
    r.part = (float *)((char *)r.head_cnt + kRunMaxHeads * sizeof(int32_t));
    if (g_run_mode == 0) {
        const int S = attn_persist_split(s, dtype, a.batch, max_pages);
        if (S > 0) return launch_attn_persist(s, dtype, r, S, st);
    }
#define FC_RL(T, DD, N, W_) launch_run_t<T, DD, N, W_>(s, r, max_pages, st)
    return FC_RUN_DISPATCH(dtype, s.D, FC_RL);
#undef FC_RL
}

}  // namespace fc
