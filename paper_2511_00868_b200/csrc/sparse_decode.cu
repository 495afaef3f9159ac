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
constexpr int kMaxPps = 256;        // max pages per split (CTA)


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

    // write state rows < G into scratch [G][D] + m/l [G]
    FC_DEVINL void store(float *wacc, float *wm, float *wl, int G, int lane) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
            l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
        }
        const int r0 = lane >> 2, c = (lane & 3) * 2;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int g = r0 + 8 * r;
            if (g < G) {
                if ((lane & 3) == 0) { wm[g] = m[r]; wl[g] = l[r]; }
#pragma unroll
                for (int i = 0; i < D / 8; ++i) {
                    wacc[g * D + i * 8 + c] = acc[i][2 * r];
                    wacc[g * D + i * 8 + c + 1] = acc[i][2 * r + 1];
                }
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

    FC_DEVINL void store(float *wacc, float *wm, float *wl, int G_, int lane) {
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            if (g >= G_) continue;
            if (lane == 0) { wm[g] = m[g]; wl[g] = l[g]; }
#pragma unroll
            for (int c = 0; c < kC; ++c) wacc[g * D + lane * kC + c] = acc[g][c];
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

template <typename T, int D, int NST>
__global__ void __launch_bounds__(kAttnWarps * 32)
attn_kernel(StoreView s, AttnArgs a) {
    using Gm = AttnGeom<T, D>;
    constexpr int NW = kAttnWarps;
    extern __shared__ __align__(128) char ring[];  // [NW][NST][page]
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ int s_page[kMaxPps];
    __shared__ int s_blk[kMaxPps];
    __shared__ float s_q[sizeof(T) == 4 ? 8 * D : 1];
    __shared__ float s_wm[NW][16], s_wl[NW][16];
    __shared__ int s_last;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int bh = blockIdx.y, c = blockIdx.x;
    const int b = bh / s.H, h = bh % s.H;
    const int G = s.G;
    const int hx = s.hix(b, a.layer, h);
    const int n_tok = s.seq_len[b] + a.extra_tokens;
    if (n_tok <= 0) return;
    const int n_pages = (n_tok + kPageSize - 1) / kPageSize;
    const int nsel = s.n_sel[hx];
    const int32_t *selrow = s.sel + (int64_t)hx * s.SELCAP;
    const int hi = nsel > 0 ? selrow[nsel - 1] : -1;
    const int n_att = a.attend_appended ? nsel + max(0, n_pages - 1 - hi) : nsel;
    const int n_splits = (n_att + a.pps - 1) / a.pps;
    if (c >= n_splits) return;
    const int j0 = c * a.pps;
    const int cnt = min(a.pps, n_att - j0);

    for (int j = tid; j < cnt; j += blockDim.x) {
        const int idx = j0 + j;
        const int page = idx < nsel ? selrow[idx] : hi + 1 + (idx - nsel);
        int blk = 0;
        if (page >= 0 && page < n_pages) blk = s.table[s.table_off(hx, page)];
        if (blk == FC_NULL_BLOCK) {  // residency violation (attention.py:101-105)
            set_error(s.err, FC_ERR_NULL_READ);
            blk = -1;
        }
        s_page[j] = page;
        s_blk[j] = blk;
    }
    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    const int64_t qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    if constexpr (sizeof(T) == 4) {
        const float *qg = reinterpret_cast<const float *>(a.q) + qoff;
        for (int i = tid; i < G * D; i += blockDim.x) s_q[i] = qg[i];
    }
    fence_mbar_init();
    __syncthreads();

    // ---- per-warp pipeline over pages j = w, w+NW, ...
    const char *pool = reinterpret_cast<const char *>(s.pool);
    char *myring = ring + (size_t)w * NST * Gm::kPageBytes;
    uint64_t *mybars = bars + w * NST;
    const int nmine = cnt > w ? (cnt - w + NW - 1) / NW : 0;
    auto issue = [&](int it) {
        const int j = w + it * NW;
        const int st = it % NST;
        const int blk = s_blk[j];
        if (blk > 0) {
            mbar_arrive_expect_tx(&mybars[st], Gm::kPageBytes);
            bulk_g2s(myring + (size_t)st * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes,
                     Gm::kPageBytes, &mybars[st]);
        } else {
            mbar_arrive_expect_tx(&mybars[st], 0);
        }
    };
    if (lane == 0)
        for (int it = 0; it < min(NST, nmine); ++it) issue(it);

    typename std::conditional<sizeof(T) == 2, Bf16Warp<D>, F32Warp<D>>::type st;
    if constexpr (sizeof(T) == 2)
        st.init(reinterpret_cast<const __nv_bfloat16 *>(a.q) + qoff, G, lane);
    else
        st.init(s_q, G, lane);

    for (int it = 0; it < nmine; ++it) {
        const int stg = it % NST;
        mbar_wait(&mybars[stg], (it / NST) & 1);
        const int j = w + it * NW;
        if (s_blk[j] > 0) {
            const int ntok = min(kPageSize, n_tok - s_page[j] * kPageSize);
            st.page(myring + (size_t)stg * Gm::kPageBytes, ntok, a.scale_log2, lane);
        }
        __syncwarp();
        if (lane == 0 && it + NST < nmine) {
            fence_proxy_async_smem();
            issue(it + NST);
        }
    }
    __syncthreads();  // ring is reused as merge scratch below

    float *wacc = reinterpret_cast<float *>(ring);  // [NW][G][D]
    for (int g = lane; g < 16; g += 32) { s_wm[w][g] = -INFINITY; s_wl[w][g] = 0.f; }
    __syncwarp();
    st.store(wacc + (size_t)w * G * D, s_wm[w], s_wl[w], G, lane);
    __syncthreads();

    // ---- merge warps of this CTA
    const bool single = (n_splits == 1);
    T *out = reinterpret_cast<T *>(a.out);
    for (int e = tid; e < G * D; e += blockDim.x) {
        const int g = e / D, i = e % D;
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) M = fmaxf(M, s_wm[ww][g]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) {
            const float f = exp2f(s_wm[ww][g] - M);
            L += s_wl[ww][g] * f;
            O += wacc[((size_t)ww * G + g) * D + i] * f;
        }
        if (single) {
            store_out<T>(out + qoff + e, O / L);
            if (i == 0 && a.lse) a.lse[(int64_t)b * s.H * G + h * G + g] = (M + log2f(L)) * 0.69314718055994531f;
        } else {
            const int64_t pbase = ((int64_t)bh * a.max_splits + c) * G + g;
            a.part_o[pbase * D + i] = O;
            if (i == 0) { a.part_ml[pbase * 2] = M; a.part_ml[pbase * 2 + 1] = L; }
        }
    }
    if (single) return;

    // ---- split-K combine in the last CTA of this head
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const int ticket = atomicAdd(&a.counters[bh], 1);
        s_last = (ticket == n_splits - 1);
        if (s_last) a.counters[bh] = 0;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (int e = tid; e < G * D; e += blockDim.x) {
        const int g = e / D, i = e % D;
        float M = -INFINITY;
        for (int cc = 0; cc < n_splits; ++cc)
            M = fmaxf(M, __ldcg(a.part_ml + (((int64_t)bh * a.max_splits + cc) * G + g) * 2));
        float L = 0.f, O = 0.f;
        for (int cc = 0; cc < n_splits; ++cc) {
            const int64_t pb = ((int64_t)bh * a.max_splits + cc) * G + g;
            const float f = exp2f(__ldcg(a.part_ml + pb * 2) - M);
            L += __ldcg(a.part_ml + pb * 2 + 1) * f;
            O += __ldcg(a.part_o + pb * D + i) * f;
        }
        store_out<T>(out + qoff + e, O / L);
        if (i == 0 && a.lse) a.lse[(int64_t)b * s.H * G + h * G + g] = (M + log2f(L)) * 0.69314718055994531f;
    }
}

// ---------------------------------------------------------------------------

template <typename T, int D, int NST>
static cudaError_t launch_attn_t(const StoreView &s, const AttnArgs &a, int batch, cudaStream_t st) {
    using Gm = AttnGeom<T, D>;
    const size_t ring = (size_t)kAttnWarps * NST * Gm::kPageBytes;
    const size_t scratch = (size_t)kAttnWarps * s.G * D * sizeof(float);
    const size_t smem = ring > scratch ? ring : scratch;
    auto kern = attn_kernel<T, D, NST>;
    static bool configured = false;  // attribute set once per instantiation
    if (!configured) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(64 * 1024 * 3));
        configured = true;
    }
    dim3 grid(a.max_splits, batch * s.H);
    kern<<<grid, kAttnWarps * 32, smem, st>>>(s, a);
    return cudaGetLastError();
}

cudaError_t launch_attn(const StoreView &s, int dtype, const AttnArgs &a, int batch, cudaStream_t st) {
    if (dtype == FC_BF16) {
        if (s.D == 128) return launch_attn_t<__nv_bfloat16, 128, 3>(s, a, batch, st);
        return launch_attn_t<__nv_bfloat16, 64, 6>(s, a, batch, st);
    }
    if (s.D == 128) return launch_attn_t<float, 128, 2>(s, a, batch, st);
    return launch_attn_t<float, 64, 3>(s, a, batch, st);
}

size_t attn_workspace_bytes(const StoreView &s, int batch, int max_splits) {
    const size_t heads = (size_t)s.B * s.H;
    (void)batch;
    return heads * sizeof(int32_t)                                   // counters
           + heads * max_splits * s.G * 2 * sizeof(float)            // part_ml
           + heads * max_splits * s.G * s.D * sizeof(float);         // part_o
}

}  // namespace fc
