// attn_persist.cu — subsystem (3), persistent per-head form: the per-layer
// attention kernel's decomposition (one head per CTA cluster, warps merged in
// shared memory, CTAs of a cluster through DSMEM — attn_kernel,
// sparse_decode.cu) looping over a RUN of consecutive layers in one launch.
//
// Reference semantics per (layer, head) are sparse_decode's
// (attention.py:85-111) with the fused update_minmax (scoring.py:59-69), as
// attn_kernel.  What the persistence buys is the layer boundary: no launch,
// the next layer's plan (attended set, physical blocks) is resolved while the
// current layer streams, and each warp's page ring runs ahead into the next
// layer, so HBM keeps streaming through the layer barrier.  Layer i+1's q and
// new token are consumed only after every CTA published layer i's outputs (a
// release/acquire grid counter) — the decoder's layer chain.
//
// Constraints (checked by the launcher): all CTAs co-resident (heads x S <=
// SMs, and enough co-resident clusters), at most 32 attended pages per warp
// per layer (one per lane), G <= 8.
#include "attn_warp.cuh"
#include <cooperative_groups.h>

namespace fc {

FC_DEVINL void p_red_release_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FC_DEVINL uint32_t p_ld_acquire(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Optional per-CTA timeline (globaltimer ns) for profiling: [grid][33][4];
// [li] = layer top, consumption start (barrier passed, q loaded),
// consumption end, outputs published; [32] = entry.  Null in production.
__device__ unsigned long long *g_persist_trace = nullptr;
FC_DEVINL unsigned long long p_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// One warp's share of one layer of its head: the head, its range of
// attended entries and (lane i) the physical block of entry j0 + i.
struct PersistPlan {
    HeadInfo hd;
    int j0, n_e, blk, last_is_last_page;
};

FC_DEVINL PersistPlan persist_plan(const StoreView &s, const RunArgs &a, int layer, int bh, int kw, int nwt,
                                   int lane) {
    PersistPlan p;
    p.hd = head_info(s, layer, a.extra_tokens, a.attend_appended, bh);
    const int n_att = p.hd.n_att;
    p.j0 = (int)((int64_t)n_att * kw / nwt);
    p.n_e = (int)((int64_t)n_att * (kw + 1) / nwt) - p.j0;
    p.blk = lane < p.n_e ? resolve_block(s, p.hd, entry_page(s, p.hd, p.j0 + lane)) : 0;
    p.last_is_last_page = p.n_e > 0 && p.j0 + p.n_e == n_att &&
                          entry_page(s, p.hd, n_att - 1) == p.hd.n_pages - 1;
    return p;
}

template <typename T, int D, int NST, int NW>
__global__ void __launch_bounds__(NW * 32, 1)
attn_persist_kernel(StoreView s, RunArgs a, int S) {
    using Gm = AttnGeom<T, D>;
    namespace cg = cooperative_groups;
    // dynamic: ring [NW][NST][page] | scratch [NW][G][D] | cstate [G][D] + m,l [2][16] | (fp32) q [G][D]
    extern __shared__ __align__(128) char dsm[];
    __shared__ __align__(8) uint64_t bars[NW * NST];
    __shared__ float s_wm[NW][16], s_wl[NW][16];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = s.G;
    const int bh = blockIdx.x / S, rank = blockIdx.x % S;
    const int nwt = S * NW, kw = rank * NW + w;
    char *myring = dsm + (size_t)w * NST * Gm::kPageBytes;
    float *scratch = reinterpret_cast<float *>(dsm + (size_t)NW * NST * Gm::kPageBytes);
    float *cstate = scratch + (size_t)NW * G * D;
    float *cm = cstate + G * D, *cl = cm + 16;
    float *s_q = cl + 16;
    uint64_t *mybars = bars + w * NST;
    const char *pool = reinterpret_cast<const char *>(s.pool);
    const int b = bh / s.H, h = bh % s.H;
    const int64_t qoff = ((int64_t)b * s.H * G + (int64_t)h * G) * D;
    uint32_t *bar = a.bar + 2 * a.l0;

    unsigned long long *trace = g_persist_trace ? g_persist_trace + (size_t)blockIdx.x * 33 * 4 : nullptr;
    if (trace && tid == 0) trace[32 * 4] = p_gtimer();
    if (tid < NW * NST) mbar_init(&bars[tid], 1);
    fence_mbar_init();
    __syncthreads();
    if (a.nl == 1) griddep_launch_dependents();
    if (a.first_dep) griddep_wait();

    bool cl_wait_pending = false;  // split cluster barrier: a deferred wait
    PersistPlan cur = persist_plan(s, a, a.l0, bh, kw, nwt, lane), nxt{};
    bool nxt_ready = false;
    int issued = 0, cons = 0, il = 0, ie = 0;  // issue pointer: layer offset (0 cur, 1 next), entry
    auto pump = [&]() {
        while (issued - cons < NST) {
            if (il == 0 && ie >= cur.n_e) {
                if (!nxt_ready) break;
                il = 1;
                ie = 0;
            }
            if (il == 1 && ie >= nxt.n_e) break;
            const int blk = __shfl_sync(0xffffffffu, il == 0 ? cur.blk : nxt.blk, ie);
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
    pump();

    typename std::conditional<sizeof(T) == 2, Bf16Attn<D>, F32Warp<D>>::type st;
    for (int li = 0; li < a.nl; ++li) {
        const int l = a.l0 + li;
        const bool tr = trace != nullptr && tid == 0 && li < 32;
        if (tr) trace[li * 4] = p_gtimer();
        if (li + 1 < a.nl) {  // plan the next layer while this one's pages are in flight
            nxt = persist_plan(s, a, l + 1, bh, kw, nwt, lane);
            nxt_ready = true;
            pump();
        }
        if (li == 0) {
            if (!a.first_dep) griddep_wait();
        } else {  // layer barrier: every CTA published layer l-1
            if (tid == 0)
                while (p_ld_acquire(bar) < (uint32_t)li * gridDim.x) __nanosleep(100);
            __syncthreads();
            if (li == 1) griddep_launch_dependents();  // every CTA is resident
        }
        const T *q_l = reinterpret_cast<const T *>(a.q) + (int64_t)li * a.q_ls;
        if constexpr (sizeof(T) == 4) {
            for (int i = tid; i < G * D; i += NW * 32) s_q[i] = reinterpret_cast<const float *>(q_l)[qoff + i];
            __syncthreads();
            st.init(s_q, G, lane);
        } else {
            st.init(q_l + qoff, G, lane);
        }
        const HeadInfo &hd = cur.hd;
        const int n_att = hd.n_att;
        TokenPatch<T, D> tp;
        const int tok_slot = (hd.n_tok - 1) % kPageSize;
        const bool has_last = cur.n_e > 0 && cur.j0 + cur.n_e == n_att;
        if (a.k_new != nullptr && has_last) {
            const int64_t nk = ((int64_t)b * s.H + h) * D;
            tp.load(s, reinterpret_cast<const T *>(a.k_new) + (int64_t)li * a.kv_ls + nk,
                    reinterpret_cast<const T *>(a.v_new) + (int64_t)li * a.kv_ls + nk, hd.hx, hd.n_pages - 1,
                    tok_slot, lane);
        }
        const int last_fill = hd.n_tok - (hd.n_pages - 1) * kPageSize;
        if (tr) trace[li * 4 + 1] = p_gtimer();
        for (int i = 0; i < cur.n_e; ++i) {
            const int blk = __shfl_sync(0xffffffffu, cur.blk, i);
            const int stg = cons % NST;
            mbar_wait(&mybars[stg], (cons / NST) & 1);
            if (blk > 0) {
                char *stage = myring + (size_t)stg * Gm::kPageBytes;
                const bool last = has_last && i == cur.n_e - 1;
                if (last && a.k_new != nullptr)
                    tp.apply(s, stage, reinterpret_cast<T *>(s.pool) + s.block_off(blk), tok_slot, hd.hx,
                             hd.n_pages - 1, lane);
                st.page(stage, last && cur.last_is_last_page ? last_fill : kPageSize, a.scale_log2, lane);
            }
            __syncwarp();
            ++cons;
            pump();
        }
        // ---- merge the warps (scratch, not the ring: it holds the next layer)
        st.finalize();
        __syncwarp();
        if (tr) trace[li * 4 + 2] = p_gtimer();
        for (int g = lane; g < 16; g += 32) { s_wm[w][g] = -INFINITY; s_wl[w][g] = 0.f; }
        __syncwarp();
        st.store_partial(scratch + (size_t)w * G * D, s_wm[w], s_wl[w], G, lane);
        __syncthreads();
        T *out = reinterpret_cast<T *>(a.out) + (int64_t)li * a.o_ls + qoff;
        float *lse = a.lse ? a.lse + (int64_t)li * a.lse_ls + (int64_t)bh * G : nullptr;
        for (int e = tid; e < G * D; e += NW * 32) {
            const int g = e / D;
            float M = -INFINITY;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) M = fmaxf(M, s_wm[ww][g]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) {
                // a CTA whose warps hold no page has M = -inf: no contribution
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
        const bool last_layer = li + 1 == a.nl;
        if (S > 1) {
            // cluster merge into rank 0.  Intermediate layers: every rank
            // arrives (release) once its state is written; only rank 0 waits
            // (acquire) and pulls the states; the others go straight on — their
            // state stays intact until rank 0 has published (the grid barrier
            // orders their next write after it).  The last layer syncs twice
            // so no rank exits while rank 0 still reads its shared memory.
            cg::cluster_group cluster = cg::this_cluster();
            if (cl_wait_pending) {
                asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
                cl_wait_pending = false;
            }
            asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
            if (rank == 0 || last_layer) {
                asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
            } else {
                cl_wait_pending = true;
            }
            if (rank == 0 && n_att > 0) {
                // every rank's row maxima / sums into local shared memory once
                // (one remote load per (rank, row)), then per element only the
                // ranks' accumulator values are read remotely
                float *s_rm = scratch;                 // [S][16] (the scratch is free again)
                float *s_rl = scratch + 16 * 16;      // [S][16]
                for (int i = tid; i < S * 16; i += NW * 32) {
                    const int r = i >> 4, g = i & 15;
                    s_rm[i] = g < G ? cluster.map_shared_rank(cm, r)[g] : -INFINITY;
                    s_rl[i] = g < G ? cluster.map_shared_rank(cl, r)[g] : 0.f;
                }
                __syncthreads();
                for (int e = tid; e < G * D; e += NW * 32) {
                    const int g = e / D;
                    float M = -INFINITY;
                    for (int r = 0; r < S; ++r) M = fmaxf(M, s_rm[r * 16 + g]);
                    float L = 0.f, O = 0.f;
#pragma unroll 8
                    for (int r = 0; r < S; ++r) {
                        const float mr = s_rm[r * 16 + g];
                        const float f = mr == -INFINITY ? 0.f : exp2f(mr - M);
                        L += s_rl[r * 16 + g] * f;
                        O += cluster.map_shared_rank(cstate, r)[e] * f;
                    }
                    out[e] = T(O / L);
                    if (lse && e % D == 0) lse[g] = (M + log2f(L)) * 0.69314718055994531f;
                }
            }
            if (last_layer) cluster.sync();  // rank 0 done reading every rank's state
        }
        if (li + 1 < a.nl) {  // publish: this CTA's outputs of layer l are written
            // every output store of the CTA precedes thread 0's release (bar.sync
            // orders them; red.release is cumulative over what it observed)
            __syncthreads();
            if (tid == 0) p_red_release_add(bar, 1u);
            if (tr) trace[li * 4 + 3] = p_gtimer();
            cur = nxt;
            nxt_ready = false;
            if (il == 1) il = 0; else { il = 0; ie = 0; }
            pump();
        }
    }
    if (a.nl > 1 && tid == 0) {  // the last CTA out resets the counters for the next launch
        __threadfence();
        if (atomicAdd(bar + 1, 1u) == gridDim.x - 1) {
            bar[0] = 0u;
            bar[1] = 0u;
        }
    }
}

// ---------------------------------------------------------------------------
// host side

template <typename T, int D, int NST, int NW>
static size_t persist_smem(const StoreView &s) {
    using Gm = AttnGeom<T, D>;
    return (size_t)NW * NST * Gm::kPageBytes + (size_t)NW * s.G * D * sizeof(float) +
           ((size_t)s.G * D + 32) * sizeof(float) + (sizeof(T) == 4 ? (size_t)s.G * D * sizeof(float) : 0);
}

static int persist_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

// cluster size for `batch` rows: the most CTAs per head that keeps every CTA
// co-resident and every warp at <= 32 pages; 0 = does not fit
template <typename T, int D, int NST, int NW>
static int persist_split_t(const StoreView &s, int batch, int max_pages) {
    if (s.G > 8) return 0;
    auto kern = attn_persist_kernel<T, D, NST, NW>;
    const size_t smem = persist_smem<T, D, NST, NW>(s);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess ||
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const int heads = batch * s.H, sms = persist_sms();
    int best = 0;
    for (int S = 1; S <= max_cluster() && (int64_t)heads * S <= sms; S *= 2) {
        if (S * NW * 32 < max_pages) continue;  // a warp holds one entry per lane
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(heads * S);
        cfg.blockDim = dim3(NW * 32);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = S;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        if (clusters >= heads) best = S;  // every cluster co-resident
    }
    return best;
}

#define FC_PERSIST_DISPATCH(dtype, D, CALL)                                             \
    ((dtype) == FC_BF16 ? ((D) == 128 ? CALL(__nv_bfloat16, 128, 3, 8) : CALL(__nv_bfloat16, 64, 6, 8)) \
                        : ((D) == 128 ? CALL(float, 128, 3, 4) : CALL(float, 64, 6, 4)))

int attn_persist_split(const StoreView &s, int dtype, int batch, int max_pages) {
#define FC_PS(T, DD, N, W) persist_split_t<T, DD, N, W>(s, batch, max_pages)
    return FC_PERSIST_DISPATCH(dtype, s.D, FC_PS);
#undef FC_PS
}

template <typename T, int D, int NST, int NW>
static cudaError_t launch_persist_t(const StoreView &s, const RunArgs &a, int S, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.batch * s.H * S);
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = persist_smem<T, D, NST, NW>(s);
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
    return cudaLaunchKernelEx(&cfg, attn_persist_kernel<T, D, NST, NW>, s, a, S);
}

cudaError_t set_persist_trace(void *p) { return cudaMemcpyToSymbol(g_persist_trace, &p, sizeof(p)); }

cudaError_t launch_attn_persist(const StoreView &s, int dtype, const RunArgs &a, int S, cudaStream_t st) {
#define FC_PL(T, DD, N, W) launch_persist_t<T, DD, N, W>(s, a, S, st)
    return FC_PERSIST_DISPATCH(dtype, s.D, FC_PL);
#undef FC_PL
}

}  // namespace fc
