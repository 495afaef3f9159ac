// store.cuh — device-side view of an fc_store and its index arithmetic.
#pragma once

#include "common.cuh"

namespace fc {

// Flat head index of (row, layer, head): rows outermost, matching the
// reference's dense (request, layer, head, logical) table (blocktable.py:120).
struct StoreView {
    int B, L, H, G, D, PS, NCAP, SELCAP, NBLK;
    void *pool;
    void *summ;
    int32_t *table;
    int32_t *seq_len;
    int32_t *sel;
    int32_t *n_sel;
    int32_t *free_stack;
    int32_t *free_top;
    int32_t *step;
    uint32_t *err;

    __host__ __device__ __forceinline__ int hix(int b, int l, int h) const {
        return (b * L + l) * H + h;
    }
    __host__ __device__ __forceinline__ int64_t table_off(int hx, int page) const {
        return (int64_t)hx * NCAP + page;
    }
    // element offset of the (min|max) summary row of a page
    __host__ __device__ __forceinline__ int64_t summ_off(int hx, int page, int which) const {
        return (((int64_t)hx * NCAP + page) * 2 + which) * D;
    }
    // element offset of a physical block
    __host__ __device__ __forceinline__ int64_t block_off(int blk) const {
        return (int64_t)blk * 2 * PS * D;
    }
};

inline StoreView make_view(const fc_store *s) {
    StoreView v;
    v.B = s->batch_cap; v.L = s->layers; v.H = s->kv_heads; v.G = s->group;
    v.D = s->head_dim; v.PS = s->page_size; v.NCAP = s->pages_cap;
    v.SELCAP = s->sel_cap; v.NBLK = s->n_blocks;
    v.pool = s->kv_pool; v.summ = s->summaries; v.table = s->table;
    v.seq_len = s->seq_len; v.sel = s->sel; v.n_sel = s->n_sel;
    v.free_stack = s->free_stack; v.free_top = s->free_top; v.step = s->step;
    v.err = s->error_word;
    return v;
}

}  // namespace fc
