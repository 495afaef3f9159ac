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
    int32_t *row_phase;           // [B] or null: row b's decode step is *step + row_phase[b]
    uint8_t *row_hold;            // [B] or null: FC_HOLD_* mode of row b at this step
    unsigned long long *stats;    // [FC_STATS_N] or null: device scoring counters

    // decode step t of row b at this step (the request's own t,
    // simulator.py:437-439): the global step shifted by the row's phase
#ifdef FC_FLAT_ONLY  // (A/B build: no per-request state, no counters)
    __device__ __forceinline__ int row_step(int step0, int) const { return step0; }
    __device__ __forceinline__ int hold_mode(int) const { return FC_HOLD_NONE; }
#else
    __device__ __forceinline__ int row_step(int step0, int b) const {
        return step0 + (row_phase ? row_phase[b] : 0);
    }
    __device__ __forceinline__ int hold_mode(int b) const { return row_hold ? row_hold[b] : FC_HOLD_NONE; }
#endif
    // stable heads of row b are due: t_b % R == 0 (rerank_due, scoring.py:196-202),
    // except while the row waits for its reload or resumes after it (its
    // selection for t_b was made at the rerank step)
    __device__ __forceinline__ bool boundary(int step0, int b, int period) const {
        const int m = hold_mode(b);
        if (m == FC_HOLD_WAIT || m == FC_HOLD_RESUME) return false;
        return row_step(step0, b) % period == 0;
    }
    // a head of row b is due: forced, unstable (every step) or at the row's
    // boundary; a row waiting for its reload scores nothing
    __device__ __forceinline__ bool head_due(int step0, int b, bool unstable_head, int period,
                                             bool force) const {
        if (force) return true;
        if (hold_mode(b) == FC_HOLD_WAIT) return false;
        return unstable_head || boundary(step0, b, period);
    }
    // row b attends and advances this step (not held for a reload)
    __device__ __forceinline__ bool decodes(int b) const {
        const int m = hold_mode(b);
        return m != FC_HOLD_WAIT && m != FC_HOLD_RERANK;
    }
    __device__ __forceinline__ void count(int which, unsigned long long n) const {
#ifndef FC_FLAT_ONLY
        if (stats && n) atomicAdd(stats + which, n);
#endif
    }

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
    v.row_phase = s->row_phase; v.row_hold = s->row_hold;
    v.stats = reinterpret_cast<unsigned long long *>(s->stats);
    return v;
}

}  // namespace fc
