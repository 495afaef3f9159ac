// capi.cu — the extern "C" boundary (include/flexicache_b200.h).  Validates
// arguments synchronously (negative status codes, mapped to the reference's
// ValueError by the Python host layer) and launches the kernels.
#include "store.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "launchers.cuh"
#include "attn_warp.cuh"

using namespace fc;

// longest head the selection handles: 12288 pages (192k tokens at page 16)
static constexpr int kMaxPagesCap = 12288;

static thread_local char g_last_error[256] = "";

static int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return FC_OK;
    std::snprintf(g_last_error, sizeof(g_last_error), "%s", cudaGetErrorString(e));
    return FC_E_CUDA;
}

static int invalid(const char *msg) {
    std::snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
    return FC_E_INVALID;
}

static int check_store(const fc_store *s) {
    if (!s) return invalid("null store");
    if (s->page_size != kPageSize) {
        std::snprintf(g_last_error, sizeof(g_last_error), "page_size %d not compiled (16 only)", s->page_size);
        return FC_E_UNSUPPORTED;
    }
    if (s->head_dim != 64 && s->head_dim != 128) {
        std::snprintf(g_last_error, sizeof(g_last_error), "head_dim %d not compiled (64, 128)", s->head_dim);
        return FC_E_UNSUPPORTED;
    }
    if (s->dtype != FC_BF16 && s->dtype != FC_F32) return invalid("dtype must be FC_BF16 or FC_F32");
    const int gmax = (s->dtype == FC_BF16 && !FC_ATTN_TOKENS_M) ? 16 : 8;  // query group = MMA N (8)
    if (s->group < 1 || s->group > gmax) {
        std::snprintf(g_last_error, sizeof(g_last_error), "group %d outside 1..%d", s->group, gmax);
        return FC_E_UNSUPPORTED;
    }
    if (s->batch_cap < 1 || s->layers < 1 || s->kv_heads < 1 || s->pages_cap < 1 || s->sel_cap < 1 ||
        s->n_blocks < 2)
        return invalid("store geometry must be positive (n_blocks >= 2)");
    if (!s->kv_pool || !s->summaries || !s->table || !s->seq_len || !s->sel || !s->n_sel ||
        !s->free_stack || !s->free_top || !s->step || !s->error_word)
        return invalid("store has a null buffer");
    return FC_OK;
}

#define FC_CHECK(x)                 \
    do {                            \
        const int _r = (x);         \
        if (_r != FC_OK) return _r; \
    } while (0)

namespace fc {
static int g_max_cluster = 16;
int max_cluster() { return g_max_cluster; }
void set_max_cluster(int n) { g_max_cluster = n <= 0 ? 16 : (n > 16 ? 16 : n); }
}  // namespace fc

extern "C" {

const char *fc_version(void) { return "flexicache-b200 0.1 sm_100a"; }
const char *fc_last_error(void) { return g_last_error; }

/* profiling hook (not part of the ABI): per-CTA globaltimer trace of the
 * attention kernel into a device buffer [grid][4] u64, or null to disable */
int fc_debug_attn_trace(void *device_buf) { return cuda_status(set_attn_trace(device_buf)); }
int fc_debug_run_trace(void *device_buf) { return cuda_status(set_run_trace(device_buf)); }
int fc_debug_persist_trace(void *device_buf) { return cuda_status(set_persist_trace(device_buf)); }
int fc_debug_score_trace(void *device_buf) { return cuda_status(set_score_trace(device_buf)); }
int fc_debug_sa_trace(void *device_buf) { return cuda_status(set_sa_trace(device_buf)); }
/* test hook: scoring kernel choice, -1 auto, 0 balanced, 1 head-aligned */
int fc_debug_score_mode(int mode) { set_score_mode(mode); return FC_OK; }
int fc_debug_max_cluster(int n) { set_max_cluster(n); return FC_OK; }
int fc_debug_score_ctas_per_sm(int n) { set_score_ctas_per_sm(n); return FC_OK; }
/* tuning hook: byte cap of the next-layer summary warm-up in fc_score_attend
 * (0 off, < 0 default 48 MiB) */
int fc_debug_summary_prefetch(long long bytes) { set_summary_prefetch_cap(bytes); return FC_OK; }
/* test hook: attention variant, 0 cluster per head (default), 1 balanced
 * all-SM variant for small head counts */
int fc_debug_attn_mode(int mode) { set_attn_mode(mode); return FC_OK; }
/* test hook: fc_sparse_decode_layers kernel, 0 per-head cluster persistent
 * kernel when it fits (default), 1 warp-balanced persistent kernel */
int fc_debug_run_mode(int mode) { set_run_mode(mode); return FC_OK; }

int fc_free_row(const fc_store *s, int row, void *stream) {
    FC_CHECK(check_store(s));
    if (row < 0 || row >= s->batch_cap) return invalid("row out of range");
    return cuda_status(launch_free_row(make_view(s), row, (cudaStream_t)stream));
}

int fc_alloc_pages(const fc_store *s, int row, int first_page, int n_pages, void *stream) {
    FC_CHECK(check_store(s));
    if (row < 0 || row >= s->batch_cap) return invalid("row out of range");
    if (first_page < 0 || n_pages < 0 || first_page + n_pages > s->pages_cap)
        return invalid("pages beyond pages_cap");
    if (n_pages == 0) return FC_OK;
    return cuda_status(launch_alloc_pages(make_view(s), row, first_page, n_pages, (cudaStream_t)stream));
}

int fc_step_advance(const fc_store *s, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (batch < 0 || batch > s->batch_cap || batch > 1024) return invalid("batch out of range");
    return cuda_status(launch_step_advance(make_view(s), batch, nullptr, 1, (cudaStream_t)stream));
}

int fc_step_advance_counted(const fc_store *s, int batch, const uint8_t *unstable, int period, void *stream) {
    FC_CHECK(check_store(s));
    if (batch < 0 || batch > s->batch_cap || batch > 1024) return invalid("batch out of range");
    if (!unstable || period < 1) return invalid("unstable flags and period >= 1 required");
    return cuda_status(launch_step_advance(make_view(s), batch, unstable, period, (cudaStream_t)stream));
}

int fc_kv_prefill(const fc_store *s, int row, int layer, const void *k, const void *v, int n_tokens,
                  void *stream) {
    FC_CHECK(check_store(s));
    if (row < 0 || row >= s->batch_cap || layer < 0 || layer >= s->layers) return invalid("row/layer out of range");
    if (!k || !v) return invalid("null k/v");
    if (n_tokens < 0 || n_tokens > s->pages_cap * s->page_size) return invalid("n_tokens beyond capacity");
    if (n_tokens == 0) return FC_OK;
    return cuda_status(launch_prefill(make_view(s), s->dtype, row, layer, k, v, n_tokens, (cudaStream_t)stream));
}

int fc_kv_append(const fc_store *s, int layer, const void *k_new, const void *v_new, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (!k_new || !v_new) return invalid("null k/v");
    if (batch == 0) return FC_OK;
    return cuda_status(launch_append(make_view(s), s->dtype, layer, k_new, v_new, batch, (cudaStream_t)stream));
}

int fc_kv_gather(const fc_store *s, int row, int layer, int head, int n_pages, void *k_out, void *v_out,
                 void *stream) {
    FC_CHECK(check_store(s));
    if (row < 0 || row >= s->batch_cap || layer < 0 || layer >= s->layers || head < 0 || head >= s->kv_heads)
        return invalid("row/layer/head out of range");
    if (n_pages < 0 || n_pages > s->pages_cap) return invalid("n_pages out of range");
    if (!k_out || !v_out) return invalid("null output");
    if (n_pages == 0) return FC_OK;
    return cuda_status(launch_gather(make_view(s), s->dtype, row, layer, head, n_pages, k_out, v_out,
                                     (cudaStream_t)stream));
}

size_t fc_score_select_workspace_size(const fc_store *s) {
    if (check_store(s) != FC_OK) return 0;
    const size_t heads = (size_t)s->batch_cap * s->kv_heads;
    return heads * s->pages_cap * sizeof(float) + heads * sizeof(int32_t);
}

int fc_score_select(const fc_store *s, int layer, const void *q, const uint8_t *unstable, int period,
                    int force_due, int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                    int32_t *counters, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (period < 1) return invalid("period must be >= 1");  // rerank_due, scoring.py:198-199
    if (topk < 1) return invalid("k must be >= 1");          // select_topk, scoring.py:174-175
    if (topk > s->sel_cap) return FC_E_CAPACITY;
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (!q || !unstable || !scores_out || !counters) return invalid("null buffer");
    if (s->pages_cap > kMaxPagesCap) return FC_E_CAPACITY;  /* block_select keys <= 48*256 */
    if (batch == 0) return FC_OK;
    const StoreView v = make_view(s);
    if (score_attend_supported(v, s->dtype, batch) > 1) {
        // small batches: a cluster of CTAs per head (the fused kernel's scoring
        // half: keys meet in rank 0's shared memory, rank 0 selects)
        AttnArgs a = {};
        a.layer = layer;
        a.out = nullptr;
        return cuda_status(launch_score_attend(v, s->dtype, layer, q, unstable, period, force_due, topk,
                                               extra_tokens, scores_out, batch, kv_prefetch ? 1 : 0, a,
                                               (cudaStream_t)stream));
    }
    return cuda_status(launch_score(v, s->dtype, layer, q, unstable, period, force_due, topk,
                                    extra_tokens, scores_out, counters, 1, batch, kv_prefetch ? 1 : 0,
                                    (cudaStream_t)stream));
}

// ring stages of the heads a scoring launch does not score: one fewer than
// the scored heads' (-1); FC_BAL_NST overrides (0: all stages; tuning knob)
static int unscored_nst() {
    static const int nst = std::getenv("FC_BAL_NST") ? std::atoi(std::getenv("FC_BAL_NST")) : -1;
    return nst;
}

int fc_score_attend_supported(const fc_store *s, int batch) {
    if (check_store(s) != FC_OK || batch < 1 || batch > s->batch_cap || s->pages_cap > kMaxPagesCap) return 0;
    return score_attend_supported(make_view(s), s->dtype, batch);
}

int fc_score_attend(const fc_store *s, int layer, const void *q, const uint8_t *unstable, int period,
                    int force_due, int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                    const void *k_new, const void *v_new, void *out, float *lse, float scale,
                    int attend_appended, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (period < 1) return invalid("period must be >= 1");  // rerank_due, scoring.py:198-199
    if (topk < 1) return invalid("k must be >= 1");          // select_topk, scoring.py:174-175
    if (topk > s->sel_cap) return FC_E_CAPACITY;
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (!q || !unstable || !scores_out || !out) return invalid("null buffer");
    if ((k_new == nullptr) != (v_new == nullptr)) return invalid("k_new and v_new go together");
    if (k_new && extra_tokens != 1) return invalid("fused append needs extra_tokens = 1");
    if (!(scale > 0.f) || !std::isfinite(scale)) return invalid("scale must be positive");
    if (s->pages_cap > kMaxPagesCap) return FC_E_CAPACITY;
    if (batch == 0) return FC_OK;
    const StoreView v = make_view(s);
    if (!score_attend_supported(v, s->dtype, batch)) {
        std::snprintf(g_last_error, sizeof(g_last_error), "fused score+attend does not fit this batch / geometry");
        return FC_E_UNSUPPORTED;
    }
    AttnArgs a = {};
    a.layer = layer; a.q = q; a.k_new = k_new; a.v_new = v_new; a.out = out; a.lse = lse;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.extra_tokens = extra_tokens; a.attend_appended = attend_appended; a.max_splits = 1; a.bal_nst = unscored_nst();
    return cuda_status(launch_score_attend(v, s->dtype, layer, q, unstable, period, force_due, topk, extra_tokens,
                                           scores_out, batch, kv_prefetch ? 1 : 0, a, (cudaStream_t)stream));
}

// balanced launch workspace: per head ready / claim / done / spare words,
// then the launch epoch and exit count, 16-byte aligned; then the chunk states
static size_t bal_flags_bytes(size_t nh) { return ((nh * 4 + 4) * sizeof(int32_t) + 15) & ~size_t(15); }

// chunks per scored head in the balanced launch (FC_BAL_CHUNKS, 2..kBalMaxSplit)
static int bal_chunks() {
    static int nc = 0;
    if (nc == 0) {
        const char *e = std::getenv("FC_BAL_CHUNKS");
        nc = e ? std::atoi(e) : kBalMaxSplit;
        nc = nc < 2 ? 2 : (nc > kBalMaxSplit ? kBalMaxSplit : nc);
    }
    return nc;
}

int fc_score_attend_balanced_supported(const fc_store *s, int batch) {
    if (check_store(s) != FC_OK || s->pages_cap > kMaxPagesCap || batch < 1 || batch > s->batch_cap) return 0;
    return score_attend_balanced_grid(make_view(s), s->dtype, batch);
}

size_t fc_score_attend_balanced_workspace_size(const fc_store *s, int batch) {
    if (check_store(s) != FC_OK || batch < 1 || batch > s->batch_cap) return 0;
    const size_t nh = (size_t)batch * s->kv_heads;
    return bal_flags_bytes(nh) + nh * kBalMaxSplit * ((size_t)s->group * s->head_dim + 32) * sizeof(float);
}

int fc_score_attend_balanced(const fc_store *s, int layer, const void *q, const uint8_t *unstable, int period,
                             int force_due, int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                             int32_t *counters, const void *k_new, const void *v_new, void *out, float *lse,
                             float scale, int attend_appended, int batch, void *stream) {
    return fc_score_attend_balanced_ws(s, layer, q, unstable, period, force_due, topk, extra_tokens, kv_prefetch,
                                       scores_out, counters, k_new, v_new, out, lse, scale, attend_appended, batch,
                                       nullptr, 0, stream);
}

int fc_score_attend_balanced_ws(const fc_store *s, int layer, const void *q, const uint8_t *unstable, int period,
                                int force_due, int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                                int32_t *counters, const void *k_new, const void *v_new, void *out, float *lse,
                                float scale, int attend_appended, int batch, void *helper_ws, size_t helper_ws_bytes,
                                void *stream) {
    FC_CHECK(check_store(s));
    if (helper_ws && helper_ws_bytes < fc_score_attend_balanced_workspace_size(s, batch))
        return FC_E_CAPACITY;
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (period < 1) return invalid("period must be >= 1");  // rerank_due, scoring.py:198-199
    if (topk < 1) return invalid("k must be >= 1");          // select_topk, scoring.py:174-175
    if (topk > s->sel_cap) return FC_E_CAPACITY;
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (!q || !unstable || !scores_out || !counters || !out) return invalid("null buffer");
    if ((k_new == nullptr) != (v_new == nullptr)) return invalid("k_new and v_new go together");
    if (k_new && extra_tokens != 1) return invalid("fused append needs extra_tokens = 1");
    if (!(scale > 0.f) || !std::isfinite(scale)) return invalid("scale must be positive");
    if (s->pages_cap > kMaxPagesCap) return FC_E_CAPACITY;
    if (batch == 0) return FC_OK;
    const StoreView v = make_view(s);
    if (!score_attend_balanced_grid(v, s->dtype, batch)) {
        std::snprintf(g_last_error, sizeof(g_last_error), "balanced score+attend does not fit this batch / geometry");
        return FC_E_UNSUPPORTED;
    }
    AttnArgs a = {};
    a.layer = layer; a.q = q; a.k_new = k_new; a.v_new = v_new; a.out = out; a.lse = lse;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.extra_tokens = extra_tokens; a.attend_appended = attend_appended; a.max_splits = 1;
    a.bal_nst = unscored_nst();
    if (helper_ws) {  // chunked attention of the scored heads (zero-initialised workspace)
        a.bal_flags = reinterpret_cast<int32_t *>(helper_ws);
        a.bal_state = reinterpret_cast<float *>(reinterpret_cast<char *>(helper_ws) +
                                                bal_flags_bytes((size_t)batch * s->kv_heads));
        a.max_splits = bal_chunks();
        static const bool nowait = std::getenv("FC_BAL_NOWAIT") != nullptr;  // (profiling knob)
        a.bal_wait = nowait ? 0 : 1;
    }
    return cuda_status(launch_score_attend_balanced(v, s->dtype, layer, q, unstable, period, force_due, topk,
                                                    extra_tokens, scores_out, counters, batch, kv_prefetch ? 1 : 0,
                                                    a, (cudaStream_t)stream));
}

int fc_score_attend_map_fits(const fc_store *s, int n_ctas, int cluster) {
    if (check_store(s) != FC_OK || s->pages_cap > kMaxPagesCap) return 0;
    return score_attend_map_fits(make_view(s), s->dtype, n_ctas, cluster);
}

int fc_score_attend_map(const fc_store *s, int layer, const void *q, const uint8_t *unstable, int period,
                        int force_due, int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                        const void *k_new, const void *v_new, void *out, float *lse, float scale,
                        int attend_appended, int batch, const int32_t *cta_map, int n_ctas, int cluster,
                        void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (period < 1) return invalid("period must be >= 1");
    if (topk < 1) return invalid("k must be >= 1");
    if (topk > s->sel_cap) return FC_E_CAPACITY;
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (!q || !unstable || !scores_out || !out || !cta_map) return invalid("null buffer");
    if ((k_new == nullptr) != (v_new == nullptr)) return invalid("k_new and v_new go together");
    if (k_new && extra_tokens != 1) return invalid("fused append needs extra_tokens = 1");
    if (!(scale > 0.f) || !std::isfinite(scale)) return invalid("scale must be positive");
    if (cluster < 2 || cluster > 16 || n_ctas < cluster || n_ctas % cluster)
        return invalid("n_ctas must be a positive multiple of cluster (2..16)");
    if (s->pages_cap > kMaxPagesCap) return FC_E_CAPACITY;
    if (batch == 0) return FC_OK;
    const StoreView v = make_view(s);
    if (!score_attend_map_fits(v, s->dtype, n_ctas, cluster)) {
        std::snprintf(g_last_error, sizeof(g_last_error), "mixed clusters do not fit this geometry");
        return FC_E_UNSUPPORTED;
    }
    AttnArgs a = {};
    a.layer = layer; a.q = q; a.k_new = k_new; a.v_new = v_new; a.out = out; a.lse = lse;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.extra_tokens = extra_tokens; a.attend_appended = attend_appended; a.max_splits = 1; a.bal_nst = unscored_nst();
    a.cta_map = cta_map; a.map_heads = batch * s->kv_heads;
    return cuda_status(launch_score_attend_map(v, s->dtype, layer, q, unstable, period, force_due, topk,
                                               extra_tokens, scores_out, kv_prefetch ? 1 : 0, a, n_ctas, cluster,
                                               (cudaStream_t)stream));
}

int fc_score_pages(const fc_store *s, int layer, const void *q, int extra_tokens, float *scores_out, int batch,
                   void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (!q || !scores_out) return invalid("null buffer");
    if (batch == 0) return FC_OK;
    static uint8_t *dummy = nullptr;  // never dereferenced when do_select == 0
    return cuda_status(launch_score(make_view(s), s->dtype, layer, q, dummy, 1, 0, 1, extra_tokens, scores_out,
                                    nullptr, 0, batch, 0, (cudaStream_t)stream));
}

int fc_select_topk(const float *scores, int stride, const int32_t *n_valid, int n_heads, int topk, int pin_last,
                   int32_t *sel_out, int32_t *n_out, void *stream) {
    if (topk < 1) return invalid("k must be >= 1");
    if (stride < 1 || n_heads < 0) return invalid("bad stride / n_heads");
    if (stride > kMaxPagesCap) return FC_E_CAPACITY;
    if (!scores || !n_valid || !sel_out || !n_out) return invalid("null buffer");
    if (n_heads == 0) return FC_OK;
    return cuda_status(launch_select(scores, stride, n_valid, n_heads, topk, pin_last, sel_out, n_out,
                                     (cudaStream_t)stream));
}

int fc_select_topk_f64(const double *scores, int n, int topk, int pin_last, uint8_t *workspace, int32_t *sel_out,
                       int32_t *n_out, void *stream) {
    if (topk < 1) return invalid("k must be >= 1");
    if (n < 0) return invalid("n must be >= 0");
    if (n > kMaxPagesCap) return FC_E_CAPACITY;
    if (!scores || !workspace || !sel_out || !n_out) return invalid("null buffer");
    if (n == 0) return cuda_status(cudaMemsetAsync(n_out, 0, sizeof(int32_t), (cudaStream_t)stream));
    return cuda_status(launch_select_f64(scores, n, topk, pin_last ? 1 : 0, workspace, sel_out, n_out,
                                         (cudaStream_t)stream));
}

size_t fc_sparse_decode_workspace_size(const fc_store *s, int batch, int max_pages, int n_ctas) {
    if (check_store(s) != FC_OK || max_pages < 1 || n_ctas < 0) return 0;
    const StoreView v = make_view(s);
    return attn_workspace_bytes(v, batch, attn_split(v, s->dtype, batch, max_pages, n_ctas));
}

int fc_sparse_decode(const fc_store *s, int layer, const void *q, const void *k_new, const void *v_new,
                     void *out, float *lse, float scale, int extra_tokens, int attend_appended,
                     int kv_prefetch, const uint8_t *early_unstable, int early_period,
                     int max_pages, int n_ctas, void *workspace, size_t ws_bytes,
                     int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (!q || !out || !workspace) return invalid("null buffer");
    if ((k_new == nullptr) != (v_new == nullptr)) return invalid("k_new and v_new go together");
    if (k_new && extra_tokens != 1) return invalid("fused append needs extra_tokens = 1");
    if (n_ctas < 0 || n_ctas > 16) return invalid("n_ctas (CTAs per head) must be in 0..16 (0 = auto)");
    if (max_pages < 1) return invalid("max_pages must be >= 1");
    if (!(scale > 0.f) || !std::isfinite(scale)) return invalid("scale must be positive");
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (early_unstable && early_period < 1) return invalid("early_period must be >= 1");
    const StoreView v = make_view(s);
    const int grid = attn_split(v, s->dtype, batch, max_pages, n_ctas);
    const size_t need = attn_workspace_bytes(v, batch, grid);
    if (ws_bytes < need) return FC_E_CAPACITY;
    if (batch == 0) return FC_OK;
    AttnArgs a;
    a.layer = layer; a.q = q; a.k_new = k_new; a.v_new = v_new; a.out = out; a.lse = lse;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.extra_tokens = extra_tokens; a.attend_appended = attend_appended; a.max_splits = grid;
    a.kv_prefetch = kv_prefetch ? 1 : 0;
    // the balanced (grid < 0) variant shares workspace partials across launches:
    // it never overlaps its predecessor
    a.early_unstable = grid > 0 ? early_unstable : nullptr;
    a.early_period = early_period;
    char *w = (char *)workspace;
    const size_t n = grid < 0 ? (size_t)(-grid) : 0;
    a.counters = (int32_t *)w;
    a.part_m = (float *)(w + ((n * sizeof(int32_t) + 255) & ~(size_t)255));
    a.part_l = a.part_m + n * 16;
    a.part_o = a.part_l + n * 16;
    return cuda_status(launch_attn(v, s->dtype, a, batch, (cudaStream_t)stream));
}

int fc_sparse_decode_layers_supported(const fc_store *s, int batch, int max_pages) {
    if (check_store(s) != FC_OK || batch < 1 || batch > s->batch_cap || max_pages < 1) return 0;
    return attn_run_supported(make_view(s), s->dtype, batch, max_pages);
}

int fc_sparse_decode_layers_split(const fc_store *s, int batch, int max_pages) {
    if (check_store(s) != FC_OK || batch < 1 || batch > s->batch_cap || max_pages < 1) return 0;
    return attn_persist_split(make_view(s), s->dtype, batch, max_pages);
}

size_t fc_sparse_decode_layers_workspace_size(const fc_store *s, int batch, int max_pages) {
    if (check_store(s) != FC_OK || max_pages < 1) return 0;
    return attn_run_workspace_bytes(make_view(s), s->dtype, batch, max_pages);
}

int fc_sparse_decode_layers(const fc_store *s, int layer_begin, int n_layers, const void *q,
                            int64_t q_layer_stride, const void *k_new, const void *v_new,
                            int64_t kv_layer_stride, void *out, int64_t out_layer_stride, float *lse,
                            int64_t lse_layer_stride, float scale, int extra_tokens, int attend_appended,
                            int first_dep, int max_pages, void *workspace, size_t ws_bytes, int batch,
                            void *stream) {
    FC_CHECK(check_store(s));
    if (n_layers < 1 || layer_begin < 0 || layer_begin + n_layers > s->layers) return invalid("layer run out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (!q || !out || !workspace) return invalid("null buffer");
    if ((k_new == nullptr) != (v_new == nullptr)) return invalid("k_new and v_new go together");
    if (k_new && extra_tokens != 1) return invalid("fused append needs extra_tokens = 1");
    if (max_pages < 1) return invalid("max_pages must be >= 1");
    if (!(scale > 0.f) || !std::isfinite(scale)) return invalid("scale must be positive");
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (n_layers > 1 && (q_layer_stride <= 0 || out_layer_stride <= 0 || (k_new && kv_layer_stride <= 0) ||
                         (lse && lse_layer_stride <= 0)))
        return invalid("layer strides must be positive for a run of several layers");
    if (batch == 0) return FC_OK;
    const StoreView v = make_view(s);
    if (!attn_run_supported(v, s->dtype, batch, max_pages)) {
        std::snprintf(g_last_error, sizeof(g_last_error), "run kernel does not fit this geometry");
        return FC_E_UNSUPPORTED;
    }
    if (ws_bytes < attn_run_workspace_bytes(v, s->dtype, batch, max_pages)) return FC_E_CAPACITY;
    RunArgs a = {};
    a.l0 = layer_begin; a.nl = n_layers;
    a.q = q; a.q_ls = q_layer_stride;
    a.k_new = k_new; a.v_new = v_new; a.kv_ls = kv_layer_stride;
    a.out = out; a.o_ls = out_layer_stride;
    a.lse = lse; a.lse_ls = lse_layer_stride;
    a.scale_log2 = scale * 1.4426950408889634f;
    a.extra_tokens = extra_tokens; a.attend_appended = attend_appended;
    a.first_dep = first_dep ? 1 : 0;
    a.batch = batch;
    return cuda_status(launch_attn_run(v, s->dtype, a, max_pages, workspace, (cudaStream_t)stream));
}

size_t fc_rerank_workspace_size(const fc_store *s) {
    if (check_store(s) != FC_OK) return 0;
    return rerank_workspace_bytes(make_view(s));
}

int fc_rerank_recycle(const fc_store *s, int layer, const int32_t *old_sel, const int32_t *n_old,
                      const uint8_t *unstable, int period, int force_due, int old_has_tail,
                      int extra_tokens, const uint8_t *slow_resident, int32_t *copies, int max_copies, int32_t *n_copies,
                      void *workspace, int batch, void *stream) {
    return fc_rerank_recycle_rows(s, layer, old_sel, n_old, unstable, period, force_due, old_has_tail, extra_tokens,
                                  slow_resident, nullptr, copies, max_copies, n_copies, workspace, batch, stream);
}

int fc_rerank_recycle_rows(const fc_store *s, int layer, const int32_t *old_sel, const int32_t *n_old,
                           const uint8_t *unstable, int period, int force_due, int old_has_tail,
                           int extra_tokens, const uint8_t *slow_resident, const uint8_t *row_skip,
                           int32_t *copies, int max_copies, int32_t *n_copies, void *workspace, int batch,
                           void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (period < 1) return invalid("period must be >= 1");
    if (!old_sel || !n_old || !unstable || !copies || !n_copies || !workspace) return invalid("null buffer");
    if (max_copies < 0) return invalid("max_copies must be >= 0");
    if (s->sel_cap > 1024) return FC_E_CAPACITY;
    if (batch == 0) return FC_OK;
    return cuda_status(launch_rerank(make_view(s), layer, old_sel, n_old, unstable, period, force_due,
                                     old_has_tail, extra_tokens, slow_resident, row_skip, copies, max_copies, n_copies,
                                     workspace, batch, (cudaStream_t)stream));
}

int fc_fetch_pages(const fc_store *s, int layer, const void *host_pages, const int32_t *copies,
                   const int32_t *n_copies, int max_copies, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (!host_pages || !copies || !n_copies) return invalid("null buffer");
    if (max_copies <= 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_fetch(make_view(s), layer, host_pages, copies, n_copies, max_copies, pb, nullptr,
                                    nullptr, nullptr, (cudaStream_t)stream));
}

int fc_fetch_pages_ctas(const fc_store *s, int layer, const void *host_pages, const int32_t *copies,
                        const int32_t *n_copies, int max_copies, int row, int max_ctas, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (!host_pages || !copies || !n_copies) return invalid("null buffer");
    if (max_ctas < 0) return invalid("max_ctas must be >= 0");
    if (row < -1 || row >= s->batch_cap) return invalid("row out of range");
    if (max_copies <= 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_fetch(make_view(s), layer, host_pages, copies, n_copies, max_copies, pb, nullptr,
                                    nullptr, nullptr, (cudaStream_t)stream, max_ctas, row));
}

int fc_fetch_pages_staged(const fc_store *s, int layer, const void *host_pages, const int32_t *copies,
                          const int32_t *n_copies, int max_copies, const int32_t *staged_map,
                          const void *staging, int32_t *n_staged_hits, void *stream) {
    FC_CHECK(check_store(s));
    if (layer < 0 || layer >= s->layers) return invalid("layer out of range");
    if (!host_pages || !copies || !n_copies || !staged_map || !staging) return invalid("null buffer");
    if (max_copies <= 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_fetch(make_view(s), layer, host_pages, copies, n_copies, max_copies, pb, staged_map,
                                    staging, n_staged_hits, (cudaStream_t)stream));
}

int fc_stage_promoted(const fc_store *s, const int32_t *pred_sel, const int32_t *pred_n, const uint8_t *unstable,
                      const uint8_t *slow_resident, const void *host_pages, int32_t *staged_map,
                      int32_t *stage_list, int32_t *stage_count, int capacity, void *staging, int batch,
                      void *stream) {
    FC_CHECK(check_store(s));
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (!pred_sel || !pred_n || !unstable || !slow_resident || !host_pages || !staged_map || !stage_list ||
        !stage_count || !staging)
        return invalid("null buffer");
    if (capacity < 1) return invalid("capacity must be >= 1");
    if (batch == 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_stage(make_view(s), pred_sel, pred_n, unstable, slow_resident, staged_map, stage_list,
                                    stage_count, capacity, host_pages, staging, pb, batch, (cudaStream_t)stream));
}

int fc_stage_plan(const fc_store *s, const int32_t *pred_sel, const int32_t *pred_n, const uint8_t *unstable,
                  const uint8_t *slow_resident, int32_t *staged_map, int32_t *stage_list, int32_t *stage_count,
                  int capacity, int batch, int pass, void *stream) {
    FC_CHECK(check_store(s));
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (!pred_sel || !pred_n || !unstable || !slow_resident || !staged_map || !stage_list || !stage_count)
        return invalid("null buffer");
    if (capacity < 1) return invalid("capacity must be >= 1");
    if (pass < 0 || pass > 3) return invalid("pass must be in 0..3");
    return cuda_status(launch_stage_plan(make_view(s), pred_sel, pred_n, unstable, slow_resident, staged_map,
                                         stage_list, stage_count, capacity, batch, pass, (cudaStream_t)stream));
}

int fc_stage_fetch(const fc_store *s, const void *host_pages, const int32_t *stage_list, const int32_t *stage_count,
                   int capacity, void *staging, int pass, void *stream) {
    FC_CHECK(check_store(s));
    if (!host_pages || !stage_list || !stage_count || !staging) return invalid("null buffer");
    if (capacity < 1) return invalid("capacity must be >= 1");
    if (pass < 0 || pass > 3) return invalid("pass must be in 0..3");
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_stage_fetch(make_view(s), host_pages, stage_list, stage_count, capacity, staging, pb,
                                          pass, (cudaStream_t)stream));
}

int fc_stage_clear(const fc_store *s, int32_t *staged_map, const int32_t *stage_list, int32_t *stage_count,
                   int capacity, void *stream) {
    FC_CHECK(check_store(s));
    if (!staged_map || !stage_list || !stage_count) return invalid("null buffer");
    if (capacity < 1) return invalid("capacity must be >= 1");
    return cuda_status(launch_stage_clear(make_view(s), staged_map, stage_list, stage_count, capacity,
                                          (cudaStream_t)stream));
}

int fc_offload_pages(const fc_store *s, void *host_pages, const int32_t *pages, int n_pages, void *stream) {
    return fc_offload_pages_ctas(s, host_pages, pages, n_pages, 0, stream);
}

int fc_offload_pages_ctas(const fc_store *s, void *host_pages, const int32_t *pages, int n_pages, int max_ctas,
                          void *stream) {
    FC_CHECK(check_store(s));
    if (!host_pages || !pages) return invalid("null buffer");
    if (n_pages < 0) return invalid("n_pages must be >= 0");
    if (max_ctas < 0) return invalid("max_ctas must be >= 0");
    if (n_pages == 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_offload(make_view(s), host_pages, pages, n_pages, pb, max_ctas,
                                      (cudaStream_t)stream));
}

int fc_offload_filled(const fc_store *s, void *host_pages, const uint8_t *unstable, uint8_t *slow_resident,
                      int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (!host_pages || !unstable) return invalid("null buffer");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    if (batch == 0) return FC_OK;
    const int pb = 2 * s->page_size * s->head_dim * (s->dtype == FC_BF16 ? 2 : 4);
    return cuda_status(launch_offload_filled(make_view(s), host_pages, unstable, slow_resident, batch, pb,
                                             (cudaStream_t)stream));
}

int fc_evict_unselected(const fc_store *s, const uint8_t *unstable, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (!unstable) return invalid("null buffer");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    return cuda_status(launch_evict_unselected(make_view(s), unstable, batch, 0, (cudaStream_t)stream));
}

int fc_evict_pages(const fc_store *s, const int32_t *pages, int n_pages, void *stream) {
    FC_CHECK(check_store(s));
    if (!pages) return invalid("null buffer");
    if (n_pages < 0) return invalid("n_pages must be >= 0");
    if (n_pages == 0) return FC_OK;
    return cuda_status(launch_evict_pages(make_view(s), pages, n_pages, (cudaStream_t)stream));
}

int fc_trace_capture(const fc_store *s, uint32_t *trace_sel, uint32_t *trace_pool, int step_base,
                     int n_slots, int topk, int extra_tokens, int batch, void *stream) {
    FC_CHECK(check_store(s));
    if (!trace_sel || !trace_pool) return invalid("null buffer");
    if (n_slots < 1) return invalid("n_slots must be >= 1");
    if (topk < 1 || topk > s->sel_cap) return invalid("topk must be in 1..sel_cap");
    if (extra_tokens < 0 || extra_tokens > 1) return invalid("extra_tokens must be 0 or 1");
    if (batch < 0 || batch > s->batch_cap) return invalid("batch out of range");
    return cuda_status(launch_trace_capture(make_view(s), trace_sel, trace_pool, step_base, n_slots, topk,
                                            extra_tokens, batch, (cudaStream_t)stream));
}

int fc_trace_overlap(const uint32_t *sel, const uint32_t *pool, int n_steps, int layers, int kv_heads,
                     int topk, const int32_t *starts, int n_windows, int window, int max_pool,
                     int32_t *inter, void *stream) {
    if (!sel || !pool || !starts || !inter) return invalid("null buffer");
    if (layers < 1 || kv_heads < 1 || topk < 1) return invalid("zero dimension");
    if (window < 2) return invalid("window must be >= 2");
    if (n_windows < 0 || window > n_steps) return invalid("window longer than the trace");
    if (max_pool < 1 || max_pool > 8 * 200 * 1024) return invalid("max_pool out of range (1..1638400)");
    if (n_windows == 0) return FC_OK;
    return cuda_status(launch_trace_overlap(sel, pool, layers, kv_heads, topk, starts, n_windows, window,
                                            max_pool, inter, (cudaStream_t)stream));
}

}  // extern "C"
