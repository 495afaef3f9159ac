// attn_warp.cuh — per-warp page attention state (bf16 tensor-core and fp32
// CUDA-core paths), the fused append, and per-head attended-set arithmetic,
// shared by the per-layer attention kernels (sparse_decode.cu) and the
// persistent multi-layer kernel (attn_run.cu).
//
// Reference semantics: _attend / sparse_decode (attention.py:67-111),
// update_minmax (scoring.py:59-69), the stable-head attended set
// (simulator.py:416-420,512).
#pragma once
#include "launchers.cuh"
#include <type_traits>
#include <cooperative_groups.h>

namespace fc {

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
            // two accumulator chains per n-tile (even / odd k-steps) halve the
            // dependent-HMMA latency of the page
            float s2[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
            const int t = (mi >> 1) * 8 + ri;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const int c = 2 * kk + (mi & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kb + t * RB + ((c ^ (t & 7)) << 4), b0, b1, b2, b3);
                if (kk & 1) {
                    mma_bf16_16816(s2[0], qa[kk], b0, b1);
                    mma_bf16_16816(s2[1], qa[kk], b2, b3);
                } else {
                    mma_bf16_16816(s[0], qa[kk], b0, b1);
                    mma_bf16_16816(s[1], qa[kk], b2, b3);
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[j][e] += s2[j][e];
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

// bf16 tensor-core path with the page's 16 tokens as the MMA M dimension and
// the query group as N (G <= 8): S^T = K q^T is 8 HMMAs per
// page at d = 128 and O^T += V^T P^T another 8 (the G-rows-as-M form above
// pads G to 16 and needs 16 + 16).  P^T reaches the B-operand layout with two
// movmatrix transposes.  Lane l holds tokens l/4 and l/4 + 8 of query
// columns 2(l%4) and 2(l%4) + 1; the running max / sum of a column are kept
// (redundantly) by the 8 lanes sharing l%4.
FC_DEVINL uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

template <int D>
struct Bf16WarpT {
    uint32_t qb[D / 16][2];
    float acc[D / 16][4];  // O^T tile i: [d = i*16 + l/4 (+8)][g = 2(l%4) + {0,1}]
    float m[2], l[2];

    FC_DEVINL void init(const __nv_bfloat16 *qrow0, int G, int lane) {
        const int g = lane >> 2, c = (lane & 3) * 2;
        const uint32_t *q = reinterpret_cast<const uint32_t *>(qrow0 + (int64_t)g * D);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
            qb[kk][0] = g < G ? q[(kk * 16 + c) / 2] : 0u;
            qb[kk][1] = g < G ? q[(kk * 16 + 8 + c) / 2] : 0u;
        }
#pragma unroll
        for (int i = 0; i < D / 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
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
        // S^T = K q^T: A = K rows (tokens) x 16 dims, two accumulator chains
        float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
        {
            const int t = (mi & 1) * 8 + ri;
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
                const int c = 2 * kk + (mi >> 1);
                uint32_t a[4];
                ldsm_x4(kb + t * RB + ((c ^ (t & 7)) << 4), a[0], a[1], a[2], a[3]);
                if (kk & 1) mma_bf16_16816(s2, a, qb[kk][0], qb[kk][1]);
                else mma_bf16_16816(s, a, qb[kk][0], qb[kk][1]);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) s[e] += s2[e];
        }
        // s[0..1]: token t0 = l/4, columns 2(l%4) + {0,1}; s[2..3]: token t0 + 8
        const int t0 = lane >> 2;
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = (t0 + (e >> 1) * 8) < ntok ? s[e] * scale_log2 : -INFINITY;
        float alpha[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {  // query column 2(l%4) + j: max over the 16 tokens (8 lanes)
            float mx = fmaxf(x[j], x[2 + j]);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            const float mn = fmaxf(m[j], mx);
            alpha[j] = exp2f(m[j] - mn);  // m = -inf on the first page -> 0
            m[j] = mn;
        }
        float p[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) p[e] = exp2f(x[e] - m[e & 1]);
#pragma unroll
        for (int j = 0; j < 2; ++j) l[j] = l[j] * alpha[j] + (p[j] + p[2 + j]);  // this lane's tokens
#pragma unroll
        for (int i = 0; i < D / 16; ++i) {
            acc[i][0] *= alpha[0]; acc[i][1] *= alpha[1];
            acc[i][2] *= alpha[0]; acc[i][3] *= alpha[1];
        }
        // P^T as the B operand (k = token, n = column): transpose the two 8x8 blocks
        const uint32_t b0 = movmatrix_t(pack_bf16x2(p[0], p[1]));  // tokens 0-7
        const uint32_t b1 = movmatrix_t(pack_bf16x2(p[2], p[3]));  // tokens 8-15
        // O^T += V^T P^T: A = V^T (16 dims x 16 tokens) via ldmatrix.trans
        {
            const int t = (mi >> 1) * 8 + ri;
#pragma unroll
            for (int i = 0; i < D / 16; ++i) {
                const int c = 2 * i + (mi & 1);
                uint32_t a[4];
                ldsm_x4_t(vb + t * RB + ((c ^ (t & 7)) << 4), a[0], a[1], a[2], a[3]);
                mma_bf16_16816(acc[i], a, b0, b1);
            }
        }
    }

    FC_DEVINL void finalize() {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            l[j] += __shfl_xor_sync(0xffffffffu, l[j], 4);
            l[j] += __shfl_xor_sync(0xffffffffu, l[j], 8);
            l[j] += __shfl_xor_sync(0xffffffffu, l[j], 16);
        }
    }

    // partial (unnormalised acc, running max m, sum l) of columns < G
    FC_DEVINL void store_partial(float *po, float *pm, float *pl, int G, int lane) {
        const int d0 = lane >> 2, gc = (lane & 3) * 2;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int g = gc + j;
            if (g < G) {
                if (d0 == 0) { pm[g] = m[j]; pl[g] = l[j]; }
#pragma unroll
                for (int i = 0; i < D / 16; ++i) {
                    po[g * D + i * 16 + d0] = acc[i][j];
                    po[g * D + i * 16 + d0 + 8] = acc[i][2 + j];
                }
            }
        }
    }

    template <typename T>
    FC_DEVINL void store_final(T *out, float *lse, int G, int lane) {
        const int d0 = lane >> 2, gc = (lane & 3) * 2;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int g = gc + j;
            if (g < G) {
                const float inv = 1.f / l[j];
#pragma unroll
                for (int i = 0; i < D / 16; ++i) {
                    out[g * D + i * 16 + d0] = T(acc[i][j] * inv);
                    out[g * D + i * 16 + d0 + 8] = T(acc[i][2 + j] * inv);
                }
                if (lse && d0 == 0) lse[g] = (m[j] + log2f(l[j])) * 0.69314718055994531f;
            }
        }
    }
};

// the engine's bf16 path: tokens as M (FC_ATTN_TOKENS_M=0 builds the
// G-rows-as-M form, kept for comparison; it also allows G up to 16)
#ifndef FC_ATTN_TOKENS_M
#define FC_ATTN_TOKENS_M 1
#endif
template <int D>
using Bf16Attn = typename std::conditional<FC_ATTN_TOKENS_M != 0, Bf16WarpT<D>, Bf16Warp<D>>::type;

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

// The same append split in two so that its loads leave the critical path:
// load() (the new token's k / v and the page's current min / max row) is
// issued as soon as the token may be read, long before the last page is
// consumed; apply() then only writes.  Result identical to patch_token.
template <typename T, int D>
struct TokenPatch {
    static constexpr int V = D / 32;
    T kv[V], vv[V], mn[V], mx[V];
    FC_DEVINL void load(const StoreView &s, const T *kn, const T *vn, int hx, int page, int slot, int lane) {
        const int i0 = lane * V;
#pragma unroll
        for (int j = 0; j < V; ++j) { kv[j] = kn[i0 + j]; vv[j] = vn[i0 + j]; }
        if (slot != 0) {
            const T *smin = reinterpret_cast<const T *>(s.summ) + s.summ_off(hx, page, 0) + i0;
            const T *smax = reinterpret_cast<const T *>(s.summ) + s.summ_off(hx, page, 1) + i0;
#pragma unroll
            for (int j = 0; j < V; ++j) { mn[j] = smin[j]; mx[j] = smax[j]; }
        }
    }
    FC_DEVINL void apply(const StoreView &s, char *stage, T *gblock, int slot, int hx, int page, int lane) {
        const int i0 = lane * V;
        T *sk = reinterpret_cast<T *>(stage) + page_elem_offset<T>(slot, i0, D);
        T *sv = reinterpret_cast<T *>(stage) + kPageSize * D + page_elem_offset<T>(slot, i0, D);
        T *gk = gblock + page_elem_offset<T>(slot, i0, D);
        T *gv = gblock + kPageSize * D + page_elem_offset<T>(slot, i0, D);
#pragma unroll
        for (int j = 0; j < V; ++j) { sk[j] = kv[j]; sv[j] = vv[j]; gk[j] = kv[j]; gv[j] = vv[j]; }
        T *smin = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 0) + i0;
        T *smax = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 1) + i0;
#pragma unroll
        for (int j = 0; j < V; ++j) {
            if (slot == 0) {
                smin[j] = kv[j];
                smax[j] = kv[j];
            } else {
                const float f = Elem<T>::to_f(kv[j]);
                smin[j] = f < Elem<T>::to_f(mn[j]) ? kv[j] : mn[j];
                smax[j] = f > Elem<T>::to_f(mx[j]) ? kv[j] : mx[j];
            }
        }
        __syncwarp();
    }
};

// Attended page count of head bh (flat row*H + head of this layer).
struct HeadInfo {
    int hx, n_tok, n_pages, nsel, hi, n_att;
};

FC_DEVINL HeadInfo head_info(const StoreView &s, int layer, int extra_tokens, int attend_appended, int bh) {
    HeadInfo hi;
    const int b = bh / s.H, h = bh % s.H;
    hi.hx = s.hix(b, layer, h);
    // (every load issued before the hold test: it must not serialise them)
    const int len = s.seq_len[b];
    hi.nsel = s.n_sel[hi.hx];
    hi.n_tok = s.decodes(b) ? len + extra_tokens : 0;  // held rows (reload pause): nothing
    hi.n_pages = hi.n_tok > 0 ? (hi.n_tok + kPageSize - 1) / kPageSize : 0;
    hi.hi = hi.nsel > 0 ? s.sel[(int64_t)hi.hx * s.SELCAP + hi.nsel - 1] : -1;
    int n_att = attend_appended ? hi.nsel + max(0, hi.n_pages - 1 - hi.hi) : hi.nsel;
    if (hi.n_tok <= 0) n_att = 0;
    hi.n_att = n_att;
    return hi;
}

FC_DEVINL HeadInfo head_info(const StoreView &s, const AttnArgs &a, int bh) {
    return head_info(s, a.layer, a.extra_tokens, a.attend_appended, bh);
}

// page (logical) of attended entry j of a head: the selection, then the pages
// appended since its last page (simulator.py:416-420)
FC_DEVINL int entry_page(const StoreView &s, const HeadInfo &hd, int j) {
    return j < hd.nsel ? s.sel[(int64_t)hd.hx * s.SELCAP + j] : hd.hi + 1 + (j - hd.nsel);
}

// physical block of a logical page; a null block is a residency violation
// (attention.py:101-105, blocktable.py:192-198): error bit, -1
FC_DEVINL int resolve_block(const StoreView &s, const HeadInfo &hd, int page) {
    int blk = 0;
    if (page >= 0 && page < hd.n_pages) blk = s.table[s.table_off(hd.hx, page)];
    if (blk == FC_NULL_BLOCK) {
        set_error(s.err, FC_ERR_NULL_READ);
        blk = -1;
    }
    return blk;
}


// Named barrier over the first n threads of the CTA (id 1..15).
FC_DEVINL void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Attention of ONE head by the first NW warps of a CTA (S = 1 form of
// attn_kernel's body, used by the fused score+attend kernel): each warp
// streams an equal contiguous range of the head's attended pages through its
// own NST-stage cp.async.bulk ring, warps merge through shared memory, the
// append is fused (TokenPatch).  Threads >= NW*32 must not call it.  ring:
// NW*NST pages of shared memory (also the merge scratch, NW*G*D floats);
// s_q: fp32 q [G][D] (fp32 only).  Every read this needs must already be
// visible (the caller waited for the previous launch / wrote sel itself).
template <typename T, int D, int NST, int NW>
FC_DEVINL int attend_head_cta(const StoreView &s, const AttnArgs &a, int bh, char *ring, uint64_t *bars,
                              float (*s_wm)[16], float (*s_wl)[16], float *s_q, int bar_id, int S = 1,
                              int rank = 0, float *cstate = nullptr, int nst = NST) {
    // nst <= NST: ring stages in use (fewer pages in flight lowers this
    // CTA's share of a saturated HBM in favour of the launch's other CTAs)
    using Gm = AttnGeom<T, D>;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    constexpr int NT = NW * 32;
    const int G = s.G;
    const HeadInfo hd = head_info(s, a, bh);
    const int n_att = hd.n_att;
    // S > 1: the head's pages are cut over the S CTAs of a cluster (rank-major)
    const int kw = rank * NW + w, nwt = S * NW;
    const int j0 = (int)((int64_t)n_att * kw / nwt);
    const int n_e = (int)((int64_t)n_att * (kw + 1) / nwt) - j0;
    const int b = bh / s.H, h = bh % s.H;
    const int64_t qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    const int last_fill = hd.n_tok - (hd.n_pages - 1) * kPageSize;
    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    fence_mbar_init();
    fence_proxy_async_smem();  // the ring held generic-proxy data before
    named_bar_sync(bar_id, NT);
    int cur_blk = 0, nxt_blk = 0;
    {
        const int j = j0 + lane;
        if (lane < n_e) cur_blk = resolve_block(s, hd, entry_page(s, hd, j));
        if (lane + 32 < n_e) nxt_blk = resolve_block(s, hd, entry_page(s, hd, j + 32));
    }
    const char *pool = reinterpret_cast<const char *>(s.pool);
    char *myring = ring + (size_t)w * NST * Gm::kPageBytes;
    uint64_t *mybars = bars + w * NST;
    int chunk = 0;
#pragma unroll
    for (int i = 0; i < NST; ++i) {
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i);
        if (lane == 0 && i < n_e && i < nst) {
            if (blk > 0) {
                mbar_arrive_expect_tx(&mybars[i], Gm::kPageBytes);
                bulk_g2s(myring + (size_t)i * Gm::kPageBytes, pool + (int64_t)blk * Gm::kPageBytes, Gm::kPageBytes,
                         &mybars[i]);
            } else {
                mbar_arrive_expect_tx(&mybars[i], 0);
            }
        }
    }
    if constexpr (sizeof(T) == 4) {
        const float *qg = reinterpret_cast<const float *>(a.q) + qoff;
        for (int i = tid; i < G * D; i += NT) s_q[i] = qg[i];
        named_bar_sync(bar_id, NT);
    }
    typename std::conditional<sizeof(T) == 2, Bf16Attn<D>, F32Warp<D>>::type st;
    if constexpr (sizeof(T) == 4) st.init(s_q, G, lane);
    else st.init(reinterpret_cast<const T *>(a.q) + qoff, G, lane);
    TokenPatch<T, D> tp;
    const int tok_slot = (hd.n_tok - 1) % kPageSize;
    const bool last_is_last_page =
        n_e > 0 && j0 + n_e == n_att && entry_page(s, hd, n_att - 1) == hd.n_pages - 1;
    if (a.k_new != nullptr && n_e > 0 && j0 + n_e == n_att) {
        const int64_t nk = ((int64_t)b * s.H + h) * D;
        tp.load(s, reinterpret_cast<const T *>(a.k_new) + nk, reinterpret_cast<const T *>(a.v_new) + nk, hd.hx,
                hd.n_pages - 1, tok_slot, lane);
    }
    int stg = 0;
    uint32_t ph = 0;
    for (int i = 0; i < n_e; ++i) {
        if (i > 0 && (i & 31) == 0) {
            cur_blk = nxt_blk;
            ++chunk;
            const int j = j0 + (chunk + 1) * 32 + lane;
            nxt_blk = (j < j0 + n_e) ? resolve_block(s, hd, entry_page(s, hd, j)) : 0;
        }
        const int blk = __shfl_sync(0xffffffffu, cur_blk, i & 31);
        const int ni = i + nst;
        const int nb_cur = __shfl_sync(0xffffffffu, cur_blk, ni & 31);
        const int nb_nxt = __shfl_sync(0xffffffffu, nxt_blk, ni & 31);
        const int nblk = (ni >> 5) == chunk ? nb_cur : nb_nxt;
        mbar_wait(&mybars[stg], ph);
        if (blk > 0) {
            char *stage = myring + (size_t)stg * Gm::kPageBytes;
            const bool last = (j0 + i == n_att - 1);
            if (last && a.k_new != nullptr)
                tp.apply(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk), tok_slot, hd.hx,
                         hd.n_pages - 1, lane);
            st.page(stage, last && last_is_last_page ? last_fill : kPageSize, a.scale_log2, lane);
        }
        __syncwarp();
        if (lane == 0 && ni < n_e) {
            if (FC_REFILL_FENCE) fence_proxy_async_smem();
            if (nblk > 0) {
                mbar_arrive_expect_tx(&mybars[stg], Gm::kPageBytes);
                bulk_g2s(myring + (size_t)stg * Gm::kPageBytes, pool + (int64_t)nblk * Gm::kPageBytes,
                         Gm::kPageBytes, &mybars[stg]);
            } else {
                mbar_arrive_expect_tx(&mybars[stg], 0);
            }
        }
        if (++stg == nst) {
            stg = 0;
            ph ^= 1u;
        }
    }
    st.finalize();
    named_bar_sync(bar_id, NT);  // every warp done with its ring: merge scratch
    if (tid < NW * NST) mbar_inval(&bars[tid]);  // (the next call initialises them again)
    float *scratch = reinterpret_cast<float *>(ring);  // [NW][G][D]
    for (int g = lane; g < 16; g += 32) { s_wm[w][g] = -INFINITY; s_wl[w][g] = 0.f; }
    __syncwarp();
    st.store_partial(scratch + (size_t)w * G * D, s_wm[w], s_wl[w], G, lane);
    named_bar_sync(bar_id, NT);
    T *out = reinterpret_cast<T *>(a.out) + qoff;
    float *lse = a.lse ? a.lse + (int64_t)bh * G : nullptr;
    if (n_att > 0) {
        for (int e = tid; e < G * D; e += NT) {
            const int g = e / D;
            float M = -INFINITY;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) M = fmaxf(M, s_wm[ww][g]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) {
                // a CTA whose warps hold no page (S > 1) has M = -inf
                const float f = M == -INFINITY ? 0.f : exp2f(s_wm[ww][g] - M);
                L += s_wl[ww][g] * f;
                O += scratch[(size_t)ww * G * D + e] * f;
            }
            if (S == 1) {
                out[e] = T(O / L);
                if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
            } else {  // this CTA's state for the cluster merge: acc [G][D] | m [16] | l [16]
                cstate[e] = O;
                if (e % D == 0) { cstate[G * D + g] = M; cstate[G * D + 16 + g] = L; }
            }
        }
    }
    return n_att;
}

// Merge of a head attended by S CTAs of one launch whose states
// (attend_head_cta's cstate layout: acc [G][D] | m [16] | l [16]) sit in
// global memory, rank r's at states + r * (G*D + 32); read through L2.
template <typename T, int D>
FC_DEVINL void merge_head_global(const StoreView &s, const AttnArgs &a, int bh, const float *states, int S, int nt) {
    const int G = s.G, GD = G * D + 32;
    const int b = bh / s.H, h = bh % s.H;
    T *out = reinterpret_cast<T *>(a.out) + ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    float *lse = a.lse ? a.lse + (int64_t)bh * G : nullptr;
    for (int e = threadIdx.x; e < G * D; e += nt) {
        const int g = e / D;
        float M = -INFINITY;
        for (int r = 0; r < S; ++r) M = fmaxf(M, __ldcg(states + (int64_t)r * GD + G * D + g));
        float L = 0.f, O = 0.f;
        for (int r = 0; r < S; ++r) {
            const float mr = __ldcg(states + (int64_t)r * GD + G * D + g);
            const float f = mr == -INFINITY ? 0.f : exp2f(mr - M);
            L += __ldcg(states + (int64_t)r * GD + G * D + 16 + g) * f;
            O += __ldcg(states + (int64_t)r * GD + e) * f;
        }
        out[e] = T(O / L);
        if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
    }
}

// Cluster merge of a head attended by S CTAs (attend_head_cta with S > 1):
// rank 0's first nt threads combine every rank's state through DSMEM and
// write the output.  Caller: a cluster barrier before and after.
template <typename T, int D>
FC_DEVINL void merge_head_cluster(const StoreView &s, const AttnArgs &a, int bh, float *cstate, int S, int nt) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int G = s.G;
    const int b = bh / s.H, h = bh % s.H;
    T *out = reinterpret_cast<T *>(a.out) + ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    float *lse = a.lse ? a.lse + (int64_t)bh * G : nullptr;
    for (int e = threadIdx.x; e < G * D; e += nt) {
        const int g = e / D;
        float M = -INFINITY;
        for (int r = 0; r < S; ++r) M = fmaxf(M, cluster.map_shared_rank(cstate, r)[G * D + g]);
        float L = 0.f, O = 0.f;
#pragma unroll 4
        for (int r = 0; r < S; ++r) {
            const float *cr = cluster.map_shared_rank(cstate, r);
            const float mr = cr[G * D + g];
            const float f = mr == -INFINITY ? 0.f : exp2f(mr - M);
            L += cr[G * D + 16 + g] * f;
            O += cr[e] * f;
        }
        out[e] = T(O / L);
        if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
    }
}

}  // namespace fc
