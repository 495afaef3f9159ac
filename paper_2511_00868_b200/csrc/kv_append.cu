// kv_append.cu — subsystem (1): paged KV writes fused with per-page key
// min/max summaries, plus the device free list that backs the block table.
//
// Reference semantics:
//   update_minmax  scoring.py:59-69   (fold one key into its page's bounds)
//   build_minmax   scoring.py:72-90   (prefill bounds, partial last page)
//   PhysicalPool   blocktable.py:28-94 (LIFO free list, null block 0)
//   allocate_pages / allocate_page_all_heads  blocktable.py:236-263
//   evict_many     blocktable.py:280-294
#include "store.cuh"
#include <cub/block/block_scan.cuh>

namespace fc {

// ---------------------------------------------------------------------------
// allocation

// One CTA.  Pops n_entries = L*H*n_pages blocks in (layer, head, page) order.
__global__ void alloc_pages_kernel(StoreView s, int row, int first_page, int n_pages) {
    const int per_head = n_pages;
    const int n_entries = s.L * s.H * per_head;
    const int top = *s.free_top;
    if (top < n_entries) {  // atomic on failure, like allocate_many (blocktable.py:62-64)
        if (threadIdx.x == 0) set_error(s.err, FC_ERR_POOL_EXHAUSTED);
        return;
    }
    for (int e = threadIdx.x; e < n_entries; e += blockDim.x) {
        const int lh = e / per_head, p = e % per_head;
        const int l = lh / s.H, h = lh % s.H;
        const int blk = s.free_stack[top - 1 - e];
        s.table[s.table_off(s.hix(row, l, h), first_page + p)] = blk;
    }
    __syncthreads();
    if (threadIdx.x == 0) *s.free_top = top - n_entries;
}

// One CTA of up to 1024 threads.  seq_len += 1 for rows [0, batch); rows that
// now start a page get it for every (layer, head), in (row, layer, head) order.
// Rows held for a reload (row_hold WAIT / RERANK) keep their length and their
// own step t_b (row_phase -= 1).  With s.stats: score_evals_naive += L*H per
// decoding row, layer_scoring_skips += its layers with no due head (needs
// `unstable`), held-row steps += 1 per held row (Metrics, simulator.py:87-131).
__global__ void step_advance_kernel(StoreView s, int batch, const uint8_t *unstable, int period) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int rows_needing[1024];
    __shared__ int s_total;
    __shared__ int s_fail;
    __shared__ int s_no_unstable;  // layers with no unstable head (skipped at a plain step)
    const int b = threadIdx.x;
    int need = 0, len = 0;
    if (s.stats && unstable) {
        if (threadIdx.x == 0) s_no_unstable = 0;
        __syncthreads();
        for (int l = threadIdx.x; l < s.L; l += blockDim.x) {
            bool any = false;
            for (int h = 0; h < s.H; ++h) any |= unstable[l * s.H + h] != 0;
            if (!any) atomicAdd(&s_no_unstable, 1);
        }
    }
    const bool active = b < batch && s.seq_len[b] >= 0;  // seq_len < 0: a free row (serving loop), left alone
    const bool held = active && !s.decodes(b);
    if (active && !held) {
        len = s.seq_len[b] + 1;
        if (len % s.PS == 0) {
            if (len / s.PS < s.NCAP) need = 1;
            else set_error(s.err, FC_ERR_PAGES_CAP);
        }
    }
    int rank, total;
    Scan(scan_tmp).ExclusiveSum(need, rank, total);
    if (need) rows_needing[rank] = b;
    const int LH = s.L * s.H;
    const int top = *s.free_top;
    if (threadIdx.x == 0) {
        s_total = total;
        s_fail = (top < total * LH);
    }
    __syncthreads();
    if (s_fail) {
        if (threadIdx.x == 0) set_error(s.err, FC_ERR_POOL_EXHAUSTED);
    } else {
        for (int e = threadIdx.x; e < s_total * LH; e += blockDim.x) {
            const int r = rows_needing[e / LH];
            const int lh = e % LH;
            const int page = (s.seq_len[r] + 1) / s.PS;  // seq_len not yet written
            const int hx = s.hix(r, lh / s.H, lh % s.H);
            s.table[s.table_off(hx, page)] = s.free_stack[top - 1 - e];
            // the new page joins the head's selection: it is attended from now
            // on (appended pages, simulator.py:463-466,512; pinned at reranks)
            const int n = s.n_sel[hx];
            if (n > 0) {
                if (n < s.SELCAP) {
                    s.sel[(int64_t)hx * s.SELCAP + n] = page;
                    s.n_sel[hx] = n + 1;
                } else {
                    set_error(s.err, FC_ERR_SEL_CAP);
                }
            }
        }
    }
    __syncthreads();
    if (active && !held) {
        s.seq_len[b] = len;
        if (s.stats) {
            s.count(FC_STAT_SCORE_EVALS_NAIVE, (unsigned long long)LH);
            // at the row's boundary every layer has a due head; otherwise the
            // layers without an unstable head score nothing
            if (unstable && !s.boundary(*s.step, b, period)) s.count(FC_STAT_LAYER_SKIPS, s_no_unstable);
        }
    }
    if (held) {
        if (s.row_phase) s.row_phase[b] -= 1;  // t_b stays: the row decodes token t_b later
        s.count(FC_STAT_HELD_ROW_STEPS, 1);
    }
    __syncthreads();  // (every thread read *s.step above)
    if (threadIdx.x == 0) {
        if (!s_fail) *s.free_top = top - s_total * LH;
        *s.step += 1;
    }
}

// Single thread: release listed pages in list order (evict_many releases its
// sorted pages one by one, blocktable.py:283-293; the host sorts the list).
__global__ void evict_pages_kernel(StoreView s, const int32_t *pages, int n) {
    int top = *s.free_top;
    for (int i = 0; i < n; ++i) {
        const int r = pages[4 * i], l = pages[4 * i + 1], h = pages[4 * i + 2], p = pages[4 * i + 3];
        const int64_t off = s.table_off(s.hix(r, l, h), p);
        const int blk = s.table[off];
        if (blk == FC_NULL_BLOCK) {
            set_error(s.err, FC_ERR_DOUBLE_EVICT);
            continue;
        }
        s.free_stack[top++] = blk;
        s.table[off] = FC_NULL_BLOCK;
    }
    *s.free_top = top;
}

// Release every page of request row `row` (all layers and heads) to the free
// list and mark the row free (seq_len = -1, empty selections): the end of a
// request in the serving loop (the reference's _finish releases its table
// row, simulator.py).  One CTA per (layer, head); blocks are pushed with
// warp-aggregated atomics (free-list order is not deterministic here).
__global__ void free_row_kernel(StoreView s, int row) {
    const int lh = blockIdx.x, l = lh / s.H, h = lh % s.H;
    const int hx = s.hix(row, l, h);
    int32_t *trow = s.table + s.table_off(hx, 0);
    const int lane = threadIdx.x & 31;
    for (int p0 = 0; p0 < s.NCAP; p0 += blockDim.x) {
        const int p = p0 + threadIdx.x;
        const int blk = p < s.NCAP ? trow[p] : FC_NULL_BLOCK;
        const bool live = blk != FC_NULL_BLOCK;
        const unsigned m = __ballot_sync(0xffffffffu, live);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(s.free_top, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (live) {
            s.free_stack[base + __popc(m & ((1u << lane) - 1u))] = blk;
            trow[p] = FC_NULL_BLOCK;
        }
    }
    if (threadIdx.x == 0) s.n_sel[hx] = 0;
    if (lh == 0 && threadIdx.x == 0) s.seq_len[row] = -1;
}

// ---------------------------------------------------------------------------
// prefill: grid (pages, H), block D threads (thread = column)

template <typename T>
__global__ void prefill_kernel(StoreView s, int row, int layer, const T *__restrict__ k,
                               const T *__restrict__ v, int n_tokens) {
    const int page = blockIdx.x, h = blockIdx.y, i = threadIdx.x;
    const int D = s.D, PS = s.PS;
    const int hx = s.hix(row, layer, h);
    const int blk = s.table[s.table_off(hx, page)];
    if (blk == FC_NULL_BLOCK) {
        if (i == 0) set_error(s.err, FC_ERR_NULL_WRITE);
        return;
    }
    T *pool = reinterpret_cast<T *>(s.pool) + s.block_off(blk);
    const int t0 = page * PS;
    const int nt = min(PS, n_tokens - t0);
    const T *kh = k + ((int64_t)h * n_tokens + t0) * D;
    const T *vh = v + ((int64_t)h * n_tokens + t0) * D;
    T kmin = kh[i], kmax = kh[i];
    float fmin = Elem<T>::to_f(kmin), fmax = fmin;
    for (int t = 0; t < nt; ++t) {
        const T kv = kh[(int64_t)t * D + i];
        pool[page_elem_offset<T>(t, i, D)] = kv;
        pool[PS * D + page_elem_offset<T>(t, i, D)] = vh[(int64_t)t * D + i];
        const float f = Elem<T>::to_f(kv);
        if (f < fmin) { fmin = f; kmin = kv; }
        if (f > fmax) { fmax = f; kmax = kv; }
    }
    T *summ = reinterpret_cast<T *>(s.summ);
    summ[s.summ_off(hx, page, 0) + i] = kmin;
    summ[s.summ_off(hx, page, 1) + i] = kmax;
}

// ---------------------------------------------------------------------------
// decode append: one warp per (row, head); lane owns D/32 consecutive columns

template <typename T, int D>
__global__ void append_kernel(StoreView s, int layer, const T *__restrict__ k_new,
                              const T *__restrict__ v_new, int batch) {
    constexpr int V = D / 32;  // elements per lane (4 or 2 for D=128/64)
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= batch * s.H) return;
    const int b = warp / s.H, h = warp % s.H;
    const int pos = s.seq_len[b];
    const int page = pos / s.PS, slot = pos % s.PS;
    if (page >= s.NCAP) {
        if (lane == 0) set_error(s.err, FC_ERR_PAGES_CAP);
        return;
    }
    const int hx = s.hix(b, layer, h);
    const int blk = s.table[s.table_off(hx, page)];
    if (blk == FC_NULL_BLOCK) {
        if (lane == 0) set_error(s.err, FC_ERR_NULL_WRITE);
        return;
    }
    const int i0 = lane * V;
    const T *kp = k_new + ((int64_t)b * s.H + h) * D + i0;
    const T *vp = v_new + ((int64_t)b * s.H + h) * D + i0;
    T kv[V], vv[V];
#pragma unroll
    for (int j = 0; j < V; ++j) { kv[j] = kp[j]; vv[j] = vp[j]; }
    T *pool = reinterpret_cast<T *>(s.pool) + s.block_off(blk);
    // the V columns of one lane stay inside one 16-byte chunk, so the swizzled
    // destination is contiguous
    T *kd = pool + page_elem_offset<T>(slot, i0, D);
    T *vd = pool + s.PS * D + page_elem_offset<T>(slot, i0, D);
#pragma unroll
    for (int j = 0; j < V; ++j) { kd[j] = kv[j]; vd[j] = vv[j]; }
    T *smin = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 0) + i0;
    T *smax = reinterpret_cast<T *>(s.summ) + s.summ_off(hx, page, 1) + i0;
    if (slot == 0) {  // empty page: sentinel +inf/-inf folded with the key (scoring.py:43-49)
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
}

// ---------------------------------------------------------------------------
// gather (readback, offload helper): grid (pages), block D threads

template <typename T>
__global__ void gather_kernel(StoreView s, int row, int layer, int head, T *k_out, T *v_out) {
    const int page = blockIdx.x, i = threadIdx.x, D = s.D, PS = s.PS;
    const int blk = s.table[s.table_off(s.hix(row, layer, head), page)];
    const T *pool = reinterpret_cast<const T *>(s.pool) + s.block_off(blk);
    for (int t = 0; t < PS; ++t) {
        const int64_t o = ((int64_t)page * PS + t) * D + i;
        if (blk == FC_NULL_BLOCK) {
            k_out[o] = T(0.0f);
            v_out[o] = T(0.0f);
        } else {
            k_out[o] = pool[page_elem_offset<T>(t, i, D)];
            v_out[o] = pool[PS * D + page_elem_offset<T>(t, i, D)];
        }
    }
}

// ---------------------------------------------------------------------------
// launchers (called from capi.cu)

cudaError_t launch_alloc_pages(const StoreView &s, int row, int first, int n, cudaStream_t st) {
    alloc_pages_kernel<<<1, 1024, 0, st>>>(s, row, first, n);
    return cudaGetLastError();
}

cudaError_t launch_step_advance(const StoreView &s, int batch, const uint8_t *unstable, int period,
                                cudaStream_t st) {
    step_advance_kernel<<<1, 1024, 0, st>>>(s, batch, unstable, period);
    return cudaGetLastError();
}

cudaError_t launch_free_row(const StoreView &s, int row, cudaStream_t st) {
    free_row_kernel<<<s.L * s.H, 256, 0, st>>>(s, row);
    return cudaGetLastError();
}

cudaError_t launch_evict_pages(const StoreView &s, const int32_t *pages, int n, cudaStream_t st) {
    evict_pages_kernel<<<1, 1, 0, st>>>(s, pages, n);
    return cudaGetLastError();
}

cudaError_t launch_prefill(const StoreView &s, int dtype, int row, int layer, const void *k,
                           const void *v, int n_tokens, cudaStream_t st) {
    dim3 grid((n_tokens + s.PS - 1) / s.PS, s.H);
    if (dtype == FC_BF16)
        prefill_kernel<__nv_bfloat16><<<grid, s.D, 0, st>>>(
            s, row, layer, (const __nv_bfloat16 *)k, (const __nv_bfloat16 *)v, n_tokens);
    else
        prefill_kernel<float><<<grid, s.D, 0, st>>>(s, row, layer, (const float *)k,
                                                    (const float *)v, n_tokens);
    return cudaGetLastError();
}

cudaError_t launch_append(const StoreView &s, int dtype, int layer, const void *k, const void *v,
                          int batch, cudaStream_t st) {
    const int warps = batch * s.H;
    const int blocks = (warps + 3) / 4;
#define FC_APPEND(T, DD) append_kernel<T, DD><<<blocks, 128, 0, st>>>(s, layer, (const T *)k, (const T *)v, batch)
    if (dtype == FC_BF16) {
        if (s.D == 128) FC_APPEND(__nv_bfloat16, 128); else FC_APPEND(__nv_bfloat16, 64);
    } else {
        if (s.D == 128) FC_APPEND(float, 128); else FC_APPEND(float, 64);
    }
#undef FC_APPEND
    return cudaGetLastError();
}

cudaError_t launch_gather(const StoreView &s, int dtype, int row, int layer, int head, int n_pages,
                          void *k_out, void *v_out, cudaStream_t st) {
    if (dtype == FC_BF16)
        gather_kernel<__nv_bfloat16><<<n_pages, s.D, 0, st>>>(
            s, row, layer, head, (__nv_bfloat16 *)k_out, (__nv_bfloat16 *)v_out);
    else
        gather_kernel<float><<<n_pages, s.D, 0, st>>>(s, row, layer, head, (float *)k_out,
                                                       (float *)v_out);
    return cudaGetLastError();
}

}  // namespace fc
