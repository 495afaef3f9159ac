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
#include <type_traits>

namespace fc {

constexpr int kAttnWarps = 4;


template <typename T, int D>
struct AttnGeom {
    static constexpr int kPageBytes = 2 * kPageSize * D * (int)sizeof(T);
    static constexpr int kHalfBytes = kPageSize * D * (int)sizeof(T);
};

// ---------------------------------------------------------------------------
// per-warp page processing

// bf16 tensor-core path.  Query rows: r0 = lane/4 and r1 = lane/4 + 8 (G<=16).
template <int D>
struct Bf16Warp {
    uint32_t qa[D / 16][4];
    float acc[D / 8][4];
    float m[2], l[2];

    FC_DEVINL void init(const __nv_bfloat16 *qrow0, int G, int lane) {
        const int r0 = lane >> 2, r1 = r0 + 8, c = (lane & 3) * 2;
        const uint32_t *q0 = reinterpret_cast<const uint32_t *>(qrow0 + (int64_t)r0 * D);
        const uint32_t *q1 = reinterpret_cast<const uint32_t *>(qrow0 + (int64_t)r1 * D);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            qa[kk][0] = r0 < G ? q0[(kk * 16 + c) / 2] : 0u;
            qa[kk][1] = r1 < G ? q1[(kk * 16 + c) / 2] : 0u;
            qa[kk][2] = r0 < G ? q0[(kk * 16 + 8 + c) / 2] : 0u;
            qa[kk][3] = r1 < G ? q1[(kk * 16 + 8 + c) / 2] : 0u;
        }
#pragma unroll
        for (int i = 0; i < D / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
        m[0] = m[1] = -INFINITY;
        l[0] = l[1] = 0.f;
    }

    FC_DEVINL void page(char *stage, int ntok, float scale_log2, int lane) {
        constexpr int RB = D * 2;  // row bytes
        const uint32_t kb = smem_u32(stage);
        const uint32_t vb = kb + kPageSize * RB;
        if (ntok < kPageSize) {  // zero V rows past the fill (P=0 there, garbage could be NaN)
            uint4 *vz = reinterpret_cast<uint4 *>(stage + kPageSize * RB + ntok * RB);
            const int n16 = (kPageSize - ntok) * RB / 16;
            for (int i = lane; i < n16; i += 32) vz[i] = make_uint4(0, 0, 0, 0);
            __syncwarp();
        }
        const int mi = lane >> 3, ri = lane & 7;
        // S = Q Kᵀ over 16 tokens: two n-tiles of 8 tokens
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        {
            const int t = (mi >> 1) * 8 + ri;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const int c = 2 * kk + (mi & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kb + t * RB + ((c ^ (t & 7)) << 4), b0, b1, b2, b3);
                mma_bf16_16816(s[0], qa[kk], b0, b1);
                mma_bf16_16816(s[1], qa[kk], b2, b3);
            }
        }
        // online softmax; C-frag: s[j][0..1] row r0, s[j][2..3] row r1,
        // token j*8 + (lane&3)*2 + {0,1}
        const int tc = (lane & 3) * 2;
        float x[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int tok = j * 8 + tc + (e & 1);
                x[j][e] = tok < ntok ? s[j][e] * scale_log2 : -INFINITY;
            }
        float alpha[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            float mx = fmaxf(fmaxf(x[0][2 * r], x[0][2 * r + 1]), fmaxf(x[1][2 * r], x[1][2 * r + 1]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float mn = fmaxf(m[r], mx);
            alpha[r] = exp2f(m[r] - mn);  // m = -inf on the first page -> 0
            m[r] = mn;
        }
        float p[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) p[j][e] = exp2f(x[j][e] - m[e >> 1]);
#pragma unroll
        for (int r = 0; r < 2; ++r)
            l[r] = l[r] * alpha[r] + (p[0][2 * r] + p[0][2 * r + 1] + p[1][2 * r] + p[1][2 * r + 1]);
#pragma unroll
        for (int i = 0; i < D / 8; ++i) {
            acc[i][0] *= alpha[0]; acc[i][1] *= alpha[0];
            acc[i][2] *= alpha[1]; acc[i][3] *= alpha[1];
        }
        uint32_t pa[4];
        pa[0] = pack_bf16x2(p[0][0], p[0][1]);
        pa[1] = pack_bf16x2(p[0][2], p[0][3]);
        pa[2] = pack_bf16x2(p[1][0], p[1][1]);
        pa[3] = pack_bf16x2(p[1][2], p[1][3]);
        // O += P V: B = V (k = token, n = column), ldmatrix.trans
        {
            const int t = (mi & 1) * 8 + ri;
#pragma unroll
            for (int dc = 0; dc < D / 16; ++dc) {
                const int c = 2 * dc + (mi >> 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vb + t * RB + ((c ^ (t & 7)) << 4), b0, b1, b2, b3);
                mma_bf16_16816(acc[2 * dc], pa, b0, b1);
                mma_bf16_16816(acc[2 * dc + 1], pa, b2, b3);
            }
        }
    }

    FC_DEVINL void finalize() {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
            l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
        }
    }

    // partial (unnormalised acc, running max m, sum l) of rows < G
    FC_DEVINL void store_partial(float *po, float *pm, float *pl, int G, int lane) {
        const int r0 = lane >> 2, c = (lane & 3) * 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int g = r0 + 8 * r;
            if (g < G) {
                if ((lane & 3) == 0) { pm[g] = m[r]; pl[g] = l[r]; }
#pragma unroll
                for (int i = 0; i < D / 8; ++i)
                    *reinterpret_cast<float2 *>(po + g * D + i * 8 + c) = make_float2(acc[i][2 * r], acc[i][2 * r + 1]);
            }
        }
    }

    template <typename T>
    FC_DEVINL void store_final(T *out, float *lse, int G, int lane) {
        const int r0 = lane >> 2, c = (lane & 3) * 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int g = r0 + 8 * r;
            if (g < G) {
                const float inv = 1.f / l[r];
#pragma unroll
                for (int i = 0; i < D / 8; ++i) {
                    out[g * D + i * 8 + c] = T(acc[i][2 * r] * inv);
                    out[g * D + i * 8 + c + 1] = T(acc[i][2 * r + 1] * inv);
                }
                if (lse && (lane & 3) == 0) lse[g] = (m[r] + log2f(l[r])) * 0.69314718055994531f;
            }
        }
    }
};

// fp32 CUDA-core path (G <= 8).  QK: lane = (token t = lane&15, half hf = lane>>4)
// with a staggered column order (conflict-free); PV: lane owns D/32 columns.
template <int D>
struct F32Warp {
    static constexpr int kC = D / 32;
    float acc[8][kC];
    float m[8], l[8];
    const float *qs;  // shared [G][D]
    int G;

    FC_DEVINL void init(const float *qsh, int g_, int) {
        qs = qsh; G = g_;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            m[g] = -INFINITY; l[g] = 0.f;
#pragma unroll
            for (int c = 0; c < kC; ++c) acc[g][c] = 0.f;
        }
    }

    FC_DEVINL void page(char *stage, int ntok, float scale_log2, int lane) {
        const float *K = reinterpret_cast<const float *>(stage);
        const float *V = K + kPageSize * D;
        const int t = lane & 15, hf = lane >> 4;
        constexpr int HALF = D / 2;
        float dot[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) dot[g] = 0.f;
        for (int j = 0; j < HALF; ++j) {
            const int i = hf * HALF + ((j + t + 16 * hf) % HALF);
            const float kv = K[t * D + i];
#pragma unroll
            for (int g = 0; g < 8; ++g)
                if (g < G) dot[g] = fmaf(qs[g * D + i], kv, dot[g]);
        }
        float p[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G) continue;
            float x = dot[g] + __shfl_xor_sync(0xffffffffu, dot[g], 16);
            x = t < ntok ? x * scale_log2 : -INFINITY;
            float mx = x;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float mn = fmaxf(m[g], mx);
            const float alpha = exp2f(m[g] - mn);
            m[g] = mn;
            p[g] = exp2f(x - mn);
            float ps = p[g];
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            l[g] = l[g] * alpha + ps;
#pragma unroll
            for (int c = 0; c < kC; ++c) acc[g][c] *= alpha;
        }
        for (int tt = 0; tt < ntok; ++tt) {
            float v[kC];
#pragma unroll
            for (int c = 0; c < kC; ++c) v[c] = V[tt * D + lane * kC + c];
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                if (g >= G) continue;
                const float pt = __shfl_sync(0xffffffffu, p[g], tt);
#pragma unroll
                for (int c = 0; c < kC; ++c) acc[g][c] = fmaf(pt, v[c], acc[g][c]);
            }
        }
    }

    FC_DEVINL void finalize() {}

    FC_DEVINL void store_partial(float *po, float *pm, float *pl, int G_, int lane) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G_) continue;
            if (lane == 0) { pm[g] = m[g]; pl[g] = l[g]; }
#pragma unroll
            for (int c = 0; c < kC; ++c) po[g * D + lane * kC + c] = acc[g][c];
        }
    }

    template <typename T>
    FC_DEVINL void store_final(T *out, float *lse, int G_, int lane) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G_) continue;
            const float inv = 1.f / l[g];
#pragma unroll
            for (int c = 0; c < kC; ++c) out[g * D + lane * kC + c] = T(acc[g][c] * inv);
            if (lse && lane == 0) lse[g] = (m[g] + log2f(l[g])) * 0.69314718055994531f;
        }
    }
};

// ---------------------------------------------------------------------------

template <typename T>
FC_DEVINL void store_out(T *p, float v);
template <>
FC_DEVINL void store_out<__nv_bfloat16>(__nv_bfloat16 *p, float v) { *p = __float2bfloat16_rn(v); }
template <>
FC_DEVINL void store_out<float>(float *p, float v) { *p = v; }

// Fused append (update_minmax, scoring.py:59-69): the warp that consumes a
// head's last page writes the new token into the staged page (after the bulk
// copy landed), into the HBM block, and folds the key into the page summary.
template <typename T, int D>
FC_DEVINL void patch_token(const StoreView &s, char *stage, T *gblock, int slot, int hx, int page,
                           const T *kn, const T *vn, int lane) {
    constexpr int V = D / 32;  // elements per lane, inside one 16-byte chunk for bf16
    const int i0 = lane * V;
    T kv[V], vv[V];
#pragma unroll
    for (int j = 0; j < V; ++j) { kv[j] = kn[i0 + j]; vv[j] = vn[i0 + j]; }
    T *sk = reinterpret_cast<T *>(stage) + page_elem_offset<T>(slot, i0, D);
    T *sv = reinterpret_cast<T *>(stage) + kPageSize * D + page_elem_offset<T>(slot, i0, D);
    T *gk = gblock + page_elem_offset<T>(slot, i0, D);
    T *gv = gblock + kPageSize * D + page_elem_offset<T>(slot, i0, D);
#pragma unroll
    for (int j = 0; j < V; ++j) { sk[j] = kv[j]; sv[j] = vv[j]; gk[j] = kv[j]; gv[j] = vv[j]; }
    T *smin = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 0) + i0;
    T *smax = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 1) + i0;
    if (slot == 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) { smin[j] = kv[j]; smax[j] = kv[j]; }
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const float f = Elem<T>::to_f(kv[j]);
            if (f < Elem<T>::to_f(smin[j])) smin[j] = kv[j];
            if (f > Elem<T>::to_f(smax[j])) smax[j] = kv[j];
        }
    }
    __syncwarp();
}

// Attended page count of head bh (flat row*H + head of this layer).
struct HeadInfo {
    int hx, n_tok, n_pages, nsel, hi, n_att;
};

FC_DEVINL HeadInfo head_info(const StoreView &s, const AttnArgs &a, int bh) {
    HeadInfo hi;
    const int b = bh / s.H, h = bh % s.H;
    hi.hx = s.hix(b, a.layer, h);
    hi.n_tok = s.seq_len[b] + a.extra_tokens;
    hi.n_pages = hi.n_tok > 0 ? (hi.n_tok + kPageSize - 1) / kPageSize : 0;
    hi.nsel = s.n_sel[hi.hx];
    hi.hi = hi.nsel > 0 ? s.sel[(int64_t)hi.hx * s.SELCAP + hi.nsel - 1] : -1;
    int n_att = a.attend_appended ? hi.nsel + max(0, hi.n_pages - 1 - hi.hi) : hi.nsel;
    if (hi.n_tok <= 0) n_att = 0;
    hi.n_att = n_att;
    return hi;
}

constexpr int kMaxHeads = 2048;     // batch*H per launch

// Optional per-CTA timeline (globaltimer ns) for profiling: [grid][4] =
// entry, first load issued, main loop done, exit.  Null in production.
__device__ unsigned long long *g_attn_trace = nullptr;

FC_DEVINL unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr int kMinPagesPerWarp = 2;
constexpr int kMaxPagesPerWarp = 32;  // one entry per lane


// Every warp is an independent worker.  The concatenation of all heads'
// attended page lists is cut into equal contiguous ranges, one per warp of
// the grid (<= 32 pages: one page per lane to resolve).  A warp streams its
// pages through a private ring of NST cp.async.bulk stages (one 8 KiB copy per
// bf16 page, completion on an mbarrier), keeps one online-softmax state per
// segment (= the part of one head inside its range), and at a segment end
// either writes the head's output (head entirely inside the range) or
// publishes a partial (m, l, acc) at slot head + global_warp — unique because
// each new segment bumps the head index, the warp index, or both — and the
// last warp to finish a head (acq_rel counter) combines its partials.  No CTA
// barrier after the prologue: warps never wait for each other.
template <typename T, int D, int NST>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_kernel(StoreView s, AttnArgs a, int n_heads) {
    using Gm = AttnGeom<T, D>;
    constexpr int NW = kAttnWarps;
    // dynamic: ring [NW][NST][page] | (fp32) q [NW][G][D] f32 | prefix [n_heads+1]
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ int s_wsum[NW];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = s.G;
    unsigned long long *trace = g_attn_trace;
    const unsigned long long t_entry = trace ? gtimer() : 0ull;
    griddep_launch_dependents();  // let the combine kernel get scheduled early (PDL)
    griddep_wait();               // selection / seq_len come from the previous launches
    char *ring = dsm;
    float *s_q = reinterpret_cast<float *>(dsm + (size_t)NW * NST * Gm::kPageBytes);
    int *s_prefix = reinterpret_cast<int *>(s_q + (sizeof(T) == 4 ? NW * G * D : 0));

    // ---- prefix of attended pages over all heads of this layer (CTA-wide, once)
    __shared__ int s_maxatt;
    {
        int carry = 0, mx = 0;
        for (int c0 = 0; c0 < n_heads; c0 += blockDim.x) {
            const int bh = c0 + tid;
            const int cnt = bh < n_heads ? head_info(s, a, bh).n_att : 0;
            mx = max(mx, cnt);
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
            if (bh < n_heads) s_prefix[bh] = before + x - cnt;
            carry += total;
            __syncthreads();
        }
        if (tid == 0) { s_prefix[n_heads] = carry; s_maxatt = 0; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        __syncthreads();
        if (lane == 0) atomicMax(&s_maxatt, mx);
    }
    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    fence_mbar_init();
    __syncthreads();

    const int total = s_prefix[n_heads];
    const int n_workers = gridDim.x * NW;
    const int gw = blockIdx.x * NW + w;
    // pages per warp: balanced, >= 2, and a head never spans more than 32
    // warps (combine_kernel reads <= 32 partials)
    const int P = max(max(kMinPagesPerWarp, (total + n_workers - 1) / n_workers), (s_maxatt + 29) / 30);
    if (blockIdx.x == 0) {  // combine plan: warps covering each head, -1 = no combine needed
        for (int bh = tid; bh < n_heads; bh += blockDim.x) {
            const int h_beg = s_prefix[bh], h_end = s_prefix[bh + 1];
            const int fw = h_beg / P, lw = h_end > h_beg ? (h_end - 1) / P : fw;
            const bool one = h_end == h_beg || (fw == lw && h_beg >= fw * P && h_end <= fw * P + P);
            a.plan[2 * bh] = one ? -1 : fw;
            a.plan[2 * bh + 1] = lw;
        }
    }
    const int start = gw * P;
    if (start >= total) return;
    const int end = min(total, start + P);
    const int n_e = end - start;  // <= 32 (grid sized on the host)

    // ---- resolve: lane e owns entry e (page -> block, head, tokens)
    int e_blk = 0, e_bh = 0, e_meta = 0;
    if (lane < n_e) {
        const int pos = start + lane;
        int lo = 0, hi = n_heads - 1;  // last head with prefix <= pos (skips empty heads)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s_prefix[mid] <= pos) lo = mid; else hi = mid - 1;
        }
        const HeadInfo hd = head_info(s, a, lo);
        const int j = pos - s_prefix[lo];
        const int page = j < hd.nsel ? s.sel[(int64_t)hd.hx * s.SELCAP + j] : hd.hi + 1 + (j - hd.nsel);
        int blk = 0;
        if (page >= 0 && page < hd.n_pages) blk = s.table[s.table_off(hd.hx, page)];
        if (blk == FC_NULL_BLOCK) {  // residency violation (attention.py:101-105)
            set_error(s.err, FC_ERR_NULL_READ);
            blk = -1;
        }
        e_blk = blk;
        e_bh = lo;
        const bool appended_here = a.k_new != nullptr && page == hd.n_pages - 1;
        e_meta = min(kPageSize, hd.n_tok - page * kPageSize) | (appended_here ? 0x10000 : 0) |
                 ((page & 0x3fff) << 17);
    }

    const char *pool = reinterpret_cast<const char *>(s.pool);
    char *myring = ring + (size_t)w * NST * Gm::kPageBytes;
    uint64_t *mybars = bars + w * NST;
    const unsigned long long t_resolved = trace ? gtimer() : 0ull;
    int trace_flags = 0;

    // prologue: the first NST loads
#pragma unroll
    for (int i = 0; i < NST; ++i) {
        const int blk = __shfl_sync(0xffffffffu, e_blk, i);
        if (lane == 0 && i < n_e) {
            if (blk > 0) {
                mbar_arrive_expect_tx(&mybars[i], Gm::kPageBytes);
                bulk_g2s(myring + (size_t)i * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes,
                         Gm::kPageBytes, &mybars[i]);
            } else {
                mbar_arrive_expect_tx(&mybars[i], 0);
            }
        }
    }

    typename std::conditional<sizeof(T) == 2, Bf16Warp<D>, F32Warp<D>>::type st;
    T *out = reinterpret_cast<T *>(a.out);
    const T *qall = reinterpret_cast<const T *>(a.q);
    float *myq = s_q + (size_t)w * G * D;
    int cur = -1;           // head of the open segment
    int64_t qoff = 0;
    HeadInfo hd{};
    for (int i = 0; i < n_e; ++i) {
        const int bh = __shfl_sync(0xffffffffu, e_bh, i);
        const int meta = __shfl_sync(0xffffffffu, e_meta, i);
        const int blk = __shfl_sync(0xffffffffu, e_blk, i);
        const int nblk = __shfl_sync(0xffffffffu, e_blk, (i + NST) & 31);
        if (bh != cur) {
            cur = bh;
            const int b = bh / s.H, h = bh % s.H;
            qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
            hd = head_info(s, a, bh);
            if constexpr (sizeof(T) == 4) {
                __syncwarp();
                for (int k = lane; k < G * D; k += 32) myq[k] = qall[qoff + k];
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
            if (meta & 0x10000) {
                const int b = bh / s.H, h = bh % s.H;
                const int64_t nk = ((int64_t)b * s.H + h) * D;
                patch_token<T, D>(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk),
                                  (hd.n_tok - 1) % kPageSize, hd.hx, (meta >> 17) & 0x3fff,
                                  reinterpret_cast<const T *>(a.k_new) + nk,
                                  reinterpret_cast<const T *>(a.v_new) + nk, lane);
            }
            st.page(stage, meta & 0xffff, a.scale_log2, lane);
        }
        __syncwarp();
        if (lane == 0 && i + NST < n_e) {
            fence_proxy_async_smem();
            if (nblk > 0) {
                mbar_arrive_expect_tx(&mybars[stg], Gm::kPageBytes);
                bulk_g2s(myring + (size_t)stg * Gm::kPageBytes, pool + (int64_t)nblk * Gm::kPageBytes,
                         Gm::kPageBytes, &mybars[stg]);
            } else {
                mbar_arrive_expect_tx(&mybars[stg], 0);
            }
        }
        // ---- segment end (last entry of the range or head change next)
        const int next_bh = __shfl_sync(0xffffffffu, e_bh, (i + 1) & 31);
        if (i + 1 == n_e || next_bh != bh) {
            st.finalize();
            const int h_beg = s_prefix[bh], h_end = s_prefix[bh + 1];
            if (h_beg >= start && h_end <= end) {  // whole head inside this warp
                st.template store_final<T>(out + qoff, a.lse ? a.lse + (int64_t)bh * G : nullptr, G, lane);
            } else {  // partial: combined by combine_kernel (ids bh + first..last warp)
                const int64_t pid = (int64_t)bh + gw;
                st.store_partial(a.part_o + pid * G * D, a.part_m + pid * 16, a.part_l + pid * 16, G, lane);
                trace_flags |= 1;
            }
        }
    }
    if (trace && lane == 0) {  // per warp: entry, resolved, done, smid | flags << 16 | n_e << 24
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        unsigned long long *tw = trace + (size_t)gw * 4;
        tw[0] = t_entry;
        tw[1] = 0;
        tw[2] = gtimer();
        tw[3] = smid | (trace_flags << 16) | ((unsigned long long)n_e << 24) | ((unsigned long long)w << 40);
    }
}

// ---------------------------------------------------------------------------
// split-K combine: one CTA per head that spans several warps (plan >= 0).
// Launched with programmatic dependent launch right behind attn_kernel; it
// waits (griddepcontrol.wait) for the partials, loads every partial's (m, l)
// in one round, then streams the accumulators with all loads independent.
template <typename T, int D>
__global__ void __launch_bounds__(128) combine_kernel(AttnArgs a, int G) {
    constexpr int MAXP = 32;
    __shared__ float s_w[16][MAXP];
    __shared__ float s_inv[16];
    griddep_wait();
    const int bh = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int fw = a.plan[2 * bh];
    if (fw < 0) return;
    const int np = a.plan[2 * bh + 1] - fw + 1;
    const int64_t p0 = (int64_t)bh + fw;
    // (m, l) of every partial: warp w handles rows g = w, w+4, ...; lane = partial
    {
        float mv[4], lv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int g = w + 4 * k;
            mv[k] = (g < G && lane < np) ? __ldcg(a.part_m + (p0 + lane) * 16 + g) : -INFINITY;
            lv[k] = (g < G && lane < np) ? __ldcg(a.part_l + (p0 + lane) * 16 + g) : 0.f;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int g = w + 4 * k;
            if (g >= G) break;
            float M = mv[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
            const float f = lane < np ? exp2f(mv[k] - M) : 0.f;
            float L = lv[k] * f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
            s_w[g][lane] = f;
            if (lane == 0) {
                s_inv[g] = 1.f / L;
                if (a.lse) a.lse[(int64_t)bh * G + g] = (M + log2f(L)) * 0.69314718055994531f;
            }
        }
    }
    __syncthreads();
    T *out = reinterpret_cast<T *>(a.out) + (int64_t)bh * G * D;  // [batch*H][G][D] == [batch][H*G][D]
    const float4 *po = reinterpret_cast<const float4 *>(a.part_o + p0 * G * D);
    const int stride4 = G * D / 4;  // float4 per partial
    for (int e4 = tid; e4 < stride4; e4 += blockDim.x) {
        const int g = (e4 * 4) / D;
        float4 v[MAXP];
#pragma unroll
        for (int p = 0; p < MAXP; ++p)  // every load issued before any use
            if (p < np) v[p] = __ldcg(po + (int64_t)p * stride4 + e4);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int p = 0; p < MAXP; ++p) {
            if (p < np) {
                const float f = s_w[g][p];
                acc.x += f * v[p].x; acc.y += f * v[p].y; acc.z += f * v[p].z; acc.w += f * v[p].w;
            }
        }
        const float inv = s_inv[g];
        T *o = out + e4 * 4;
        o[0] = T(acc.x * inv); o[1] = T(acc.y * inv); o[2] = T(acc.z * inv); o[3] = T(acc.w * inv);
    }
}

// ---------------------------------------------------------------------------

template <typename T, int D, int NST>
static size_t attn_smem(const StoreView &s, int n_heads) {
    using Gm = AttnGeom<T, D>;
    return (size_t)kAttnWarps * NST * Gm::kPageBytes +
           (size_t)(sizeof(T) == 4 ? kAttnWarps : 0) * s.G * D * sizeof(float) +
           (size_t)(n_heads + 1) * sizeof(int);
}

template <typename T, int D, int NST>
static int attn_ctas_per_sm_t(const StoreView &s, int n_heads) {
    const size_t smem = attn_smem<T, D, NST>(s, n_heads);
    auto kern = attn_kernel<T, D, NST>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kAttnWarps * 32, smem);
    return occ < 1 ? 1 : occ;
}

#define FC_ATTN_DISPATCH(dtype, D, CALL)                                        \
    ((dtype) == FC_BF16 ? ((D) == 128 ? CALL(__nv_bfloat16, 128, 3) : CALL(__nv_bfloat16, 64, 6)) \
                        : ((D) == 128 ? CALL(float, 128, 2) : CALL(float, 64, 3)))

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

// One full wave of CTAs (occupancy x SMs), more if a warp would own more than
// kMaxPagesPerWarp pages.
int attn_grid(const StoreView &s, int dtype, int batch, int max_pages, int n_ctas) {
    if (n_ctas > 0) return n_ctas;
    const int n_heads = batch * s.H;
#define FC_OCC(T, DD, N) attn_ctas_per_sm_t<T, DD, N>(s, n_heads)
    const int occ = FC_ATTN_DISPATCH(dtype, s.D, FC_OCC);
#undef FC_OCC
    const int64_t bound = (int64_t)n_heads * max_pages;
    const int64_t wave = (int64_t)occ * num_sms();
    const int64_t per_cta = (int64_t)kMaxPagesPerWarp * kAttnWarps;
    const int64_t need = (bound + per_cta - 1) / per_cta;
    return (int)(need > wave ? need : wave);
}

template <typename T, int D, int NST>
static cudaError_t launch_attn_t(const StoreView &s, const AttnArgs &a, int batch, cudaStream_t st) {
    const int n_heads = batch * s.H;
    const size_t smem = attn_smem<T, D, NST>(s, n_heads);
    cudaError_t e = launch_pdl(attn_kernel<T, D, NST>, dim3(a.max_splits), dim3(kAttnWarps * 32), smem, st,
                               s, a, n_heads);
    if (e != cudaSuccess) return e;
    return launch_pdl(combine_kernel<T, D>, dim3(n_heads), dim3(128), 0, st, a, s.G);
}

cudaError_t set_attn_trace(void *p) {
    return cudaMemcpyToSymbol(g_attn_trace, &p, sizeof(p));
}

cudaError_t launch_attn(const StoreView &s, int dtype, const AttnArgs &a, int batch, cudaStream_t st) {
    if (batch * s.H > kMaxHeads) return cudaErrorInvalidValue;
    if (dtype == FC_BF16) {
        if (s.D == 128) return launch_attn_t<__nv_bfloat16, 128, 3>(s, a, batch, st);
        return launch_attn_t<__nv_bfloat16, 64, 6>(s, a, batch, st);
    }
    if (s.D == 128) return launch_attn_t<float, 128, 2>(s, a, batch, st);
    return launch_attn_t<float, 64, 3>(s, a, batch, st);
}

size_t attn_workspace_bytes(const StoreView &s, int batch, int n_ctas) {  // n_ctas = launched grid
    const size_t heads = (size_t)s.B * s.H;
    const size_t parts = heads + (size_t)n_ctas * kAttnWarps;  // partial ids h + global warp
    (void)batch;
    return ((2 * heads * sizeof(int32_t) + 255) & ~(size_t)255) + parts * 16 * 2 * sizeof(float) +
           parts * s.G * s.D * sizeof(float);
}

}  // namespace fc
