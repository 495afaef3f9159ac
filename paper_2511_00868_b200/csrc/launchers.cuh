// launchers.cuh — host-side launcher declarations shared by the .cu files.
#pragma once
#include "store.cuh"

namespace fc {
// largest cluster (CTAs per head) the automatic splits may choose (16; a
// test hook pins it so differently sized launches split heads alike)
int max_cluster();
void set_max_cluster(int n);
struct AttnArgs {
    int layer;
    const void *q;
    const void *k_new;    // fused append: [batch][H][D] or null
    const void *v_new;
    void *out;
    float *lse;
    float scale_log2;
    int extra_tokens;
    int attend_appended;
    int kv_prefetch;      // stage KV pages before the previous launch completes
    const uint8_t *early_unstable;  // [L][H]: heads not due this step skip the wait
    int early_period;
    int max_splits;       // CTAs per head (cluster size S)
    int32_t *counters;    // [B_cap*H] partials published per head (zeroed once, self-resetting)
    float *part_m;        // [parts][16]
    float *part_l;        // [parts][16]
    float *part_o;
    // fc_score_attend_map: per CTA a head (bit 30: attends it alone, as a
    // cluster of one) or -1 (idle); null = CTA i / S attends head i / S
    const int32_t *cta_map;
    int map_heads;        // batch * H: bound of the map's head indices
    // fc_score_attend: CTAs of heads not scored this step, once their pages
    // are attended, warm L2 with the next layer's due summaries (the scored
    // CTAs of that layer then stream them from L2) when those are at most
    // this many bytes; 0 = off (set by the launcher)
    int64_t pf_cap;
    // fc_score_attend_balanced: the scored heads' attention cut into
    // max_splits chunks claimed by any CTA with no work left (null = off):
    // per head ready / claim / done / spare words [4][batch*H], the launch
    // epoch and exit count, and the chunk states [batch*H][kBalMaxSplit][G*D + 32]
    int32_t *bal_flags;
    float *bal_state;
    int bal_nst;          // balanced launch: ring stages of the heads that are not scored (-1: NST - 1, 0: all)
    int bal_wait;         // balanced launch: CTAs with no work wait for selections still pending
    int compact_select;   // fc_score_attend: rolled-loop select (block_select_compact)
};
constexpr int kBalMaxSplit = 4;  // chunks of one scored head's attention (balanced launch)

// persistent multi-layer attention (attn_run.cu)
struct RunArgs {
    int l0, nl;            // layers [l0, l0 + nl)
    const void *q;         // layer l0 + i at q + i * q_ls elements: [batch][H*G][D]
    int64_t q_ls;
    const void *k_new;     // [batch][H][D] per layer (kv_ls apart) or null
    const void *v_new;
    int64_t kv_ls;
    void *out;
    int64_t o_ls;
    float *lse;            // [batch*H*G] per layer (lse_ls apart) or null
    int64_t lse_ls;
    float scale_log2;
    int extra_tokens, attend_appended;
    int first_dep;         // the previous launch writes layer l0's selection / table
    int batch;
    int min_pages, maxr;   // set by the launcher
    uint32_t *bar;         // workspace: [L][2] barrier / exit counters (self-resetting)
    int32_t *head_cnt;     // workspace: per-head part counters (self-resetting)
    float *part;           // workspace: [warps][2][G*D + 32]
};
int attn_run_supported(const StoreView &, int, int, int);
size_t attn_run_workspace_bytes(const StoreView &, int, int, int);
cudaError_t launch_attn_run(const StoreView &, int, const RunArgs &, int, void *, cudaStream_t);
int attn_persist_split(const StoreView &, int, int, int);
cudaError_t launch_attn_persist(const StoreView &, int, const RunArgs &, int, cudaStream_t);

cudaError_t launch_alloc_pages(const StoreView &, int, int, int, cudaStream_t);
cudaError_t launch_step_advance(const StoreView &, int, const uint8_t *, int, cudaStream_t);
cudaError_t launch_free_row(const StoreView &, int, cudaStream_t);
cudaError_t launch_evict_pages(const StoreView &, const int32_t *, int, cudaStream_t);
cudaError_t launch_prefill(const StoreView &, int, int, int, const void *, const void *, int, cudaStream_t);
cudaError_t launch_append(const StoreView &, int, int, const void *, const void *, int, cudaStream_t);
cudaError_t launch_gather(const StoreView &, int, int, int, int, int, void *, void *, cudaStream_t);
cudaError_t launch_score(const StoreView &, int, int, const void *, const uint8_t *, int, int, int, int,
                         float *, int32_t *, int, int, int, cudaStream_t);
int score_attend_supported(const StoreView &, int, int);
int score_attend_map_fits(const StoreView &, int, int, int);
cudaError_t launch_score_attend_map(const StoreView &, int, int, const void *, const uint8_t *, int, int, int, int,
                                    float *, int, const AttnArgs &, int, int, cudaStream_t);
cudaError_t launch_score_attend(const StoreView &, int, int, const void *, const uint8_t *, int, int, int, int,
                                float *, int, int, const AttnArgs &, cudaStream_t);
int score_attend_balanced_grid(const StoreView &, int, int);
cudaError_t launch_score_attend_balanced(const StoreView &, int, int, const void *, const uint8_t *, int, int, int, int,
                                         float *, int32_t *, int, int, const AttnArgs &, cudaStream_t);
cudaError_t launch_select(const float *, int, const int32_t *, int, int, int, int32_t *, int32_t *,
                          cudaStream_t);
cudaError_t launch_attn(const StoreView &, int, const AttnArgs &, int, cudaStream_t);
size_t attn_workspace_bytes(const StoreView &, int, int);
cudaError_t set_attn_trace(void *);
cudaError_t set_run_trace(void *);
cudaError_t set_persist_trace(void *);
cudaError_t set_score_trace(void *);
cudaError_t set_sa_trace(void *);
void set_score_mode(int);
void set_score_ctas_per_sm(int);
void set_summary_prefetch_cap(int64_t bytes);  // < 0: default
void set_attn_mode(int);
void set_run_mode(int);
cudaError_t launch_trace_capture(const StoreView &, uint32_t *, uint32_t *, int, int, int, int, int, cudaStream_t);
cudaError_t launch_trace_overlap(const uint32_t *, const uint32_t *, int, int, int, const int32_t *, int, int,
                                 int, int32_t *, cudaStream_t);
int attn_split(const StoreView &, int, int, int, int);
size_t rerank_workspace_bytes(const StoreView &);
cudaError_t launch_rerank(const StoreView &, int, const int32_t *, const int32_t *, const uint8_t *, int,
                          int, int, int, const uint8_t *, const uint8_t *, int32_t *, int, int32_t *, void *, int,
                          cudaStream_t);
cudaError_t launch_fetch(const StoreView &, int, const void *, const int32_t *, const int32_t *, int, int,
                         const int32_t *, const void *, int32_t *, cudaStream_t, int max_ctas = 0, int row = -1);
cudaError_t launch_stage(const StoreView &, const int32_t *, const int32_t *, const uint8_t *, const uint8_t *,
                         int32_t *, int32_t *, int32_t *, int, const void *, void *, int, int, cudaStream_t);
cudaError_t launch_stage_plan(const StoreView &, const int32_t *, const int32_t *, const uint8_t *, const uint8_t *,
                              int32_t *, int32_t *, int32_t *, int, int, int, cudaStream_t);
cudaError_t launch_stage_fetch(const StoreView &, const void *, const int32_t *, const int32_t *, int, void *, int,
                               int, cudaStream_t);
cudaError_t launch_stage_clear(const StoreView &, int32_t *, const int32_t *, int32_t *, int, cudaStream_t);
cudaError_t launch_offload(const StoreView &, void *, const int32_t *, int, int, int, cudaStream_t);
cudaError_t launch_offload_filled(const StoreView &, void *, const uint8_t *, uint8_t *, int, int, cudaStream_t);
cudaError_t launch_evict_unselected(const StoreView &, const uint8_t *, int, int, cudaStream_t);

cudaError_t launch_select_f64(const double *, int, int, int, uint8_t *, int32_t *, int32_t *, cudaStream_t);
}  // namespace fc
