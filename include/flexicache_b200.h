/*
 * flexicache_b200.h — C ABI of the B200-native FlexiCache per-decode-step KV
 * hot path (sm_100a).  Drop-in for the reference's Python hot-path calls
 * (tierkv, /root/reference/pkg/src/tierkv); each entry point names the
 * reference function(s) it replaces.
 *
 * Conventions
 *  - The library never allocates device memory.  Every buffer is owned by the
 *    caller (PyTorch on the host side) and passed as a raw device pointer in
 *    an fc_store descriptor or as an argument with explicit sizes.
 *  - Every call is asynchronous on the given cudaStream_t (passed as void*)
 *    and returns an int status: FC_OK or a negative FC_E* code for
 *    synchronous argument errors.  Device-side invariant violations (read of
 *    the null block, pool exhaustion, capacity overflow) set sticky bits in
 *    store->error_word, which the host wrapper inspects and maps to the
 *    reference's exception types (errors.py:26,30).
 *  - Stateless and reentrant: safe on distinct streams with distinct buffers.
 *  - Layouts are documented in DESIGN.md §3.  Elements are bf16 (FC_BF16) or
 *    fp32 (FC_F32).  Page size is 16 tokens; head_dim is 64 or 128.
 */
#ifndef FLEXICACHE_B200_H
#define FLEXICACHE_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define FC_OK               0
#define FC_E_INVALID      (-1)  /* bad argument: maps to ValueError            */
#define FC_E_UNSUPPORTED  (-2)  /* geometry not compiled (d, ps, G): ValueError */
#define FC_E_CUDA         (-3)  /* CUDA launch/runtime error                     */
#define FC_E_CAPACITY     (-4)  /* workspace / capacity too small                */

/* element types */
#define FC_BF16 0
#define FC_F32  1

/* sticky device error bits in *error_word */
#define FC_ERR_POOL_EXHAUSTED   1u  /* PoolExhausted      (blocktable.py:52-54)      */
#define FC_ERR_NULL_READ        2u  /* ConsistencyError   (blocktable.py:192-198,
                                                           attention.py:101-105)     */
#define FC_ERR_NULL_WRITE       4u  /* append into a page with no block              */
#define FC_ERR_PAGES_CAP        8u  /* logical page beyond pages_cap                 */
#define FC_ERR_SEL_CAP         16u  /* selection longer than sel_cap                 */
#define FC_ERR_DOUBLE_EVICT    32u  /* ConsistencyError   (blocktable.py:319-322)    */
#define FC_ERR_WRITE_TWICE     64u  /* ConsistencyError   (tiering.py:105-110 ledger) */
#define FC_ERR_TRACE_SHORT    128u  /* trace capture: a selection shorter than K      */
#define FC_ERR_RUN_RANGE      256u  /* fc_sparse_decode_layers: warp range overflow (sizing bug) */

#define FC_NULL_BLOCK 0             /* blocktable.py:25 */

/*
 * Device KV store: the batched, GPU-resident form of the reference's
 * per-(request, layer, head) state — PhysicalPool + BlockTable
 * (blocktable.py:28-440), MinMaxCache (scoring.py:114-139) and the per-head
 * TopKSet (scoring.py:142-161).
 */
typedef struct fc_store {
    int32_t batch_cap;   /* B_cap request rows                                   */
    int32_t layers;      /* L                                                    */
    int32_t kv_heads;    /* H_kv per layer                                       */
    int32_t group;       /* G = H_q / H_kv (1..8)                                */
    int32_t head_dim;    /* d: 64 or 128                                         */
    int32_t page_size;   /* ps: 16                                               */
    int32_t pages_cap;   /* N_cap logical pages per (row, layer, head)           */
    int32_t sel_cap;     /* entries per selection row                            */
    int32_t dtype;       /* FC_BF16 or FC_F32                                    */
    int32_t n_blocks;    /* physical blocks incl. the null block 0               */
    void    *kv_pool;    /* [n_blocks][2][ps][d] elements (K rows then V rows)   */
    void    *summaries;  /* [B_cap][L][H][N_cap][2][d] elements (min, max rows)  */
    int32_t *table;      /* [B_cap][L][H][N_cap] physical block, 0 = not resident*/
    int32_t *seq_len;    /* [B_cap] tokens stored in every layer                 */
    int32_t *sel;        /* [B_cap][L][H][sel_cap] ascending logical pages       */
    int32_t *n_sel;      /* [B_cap][L][H]; 0 = no selection yet (attend all)     */
    int32_t *free_stack; /* [n_blocks] LIFO free list, top at free_top-1         */
    int32_t *free_top;   /* [1]                                                  */
    int32_t *step;       /* [1] decode step t of the upcoming step (1-based)     */
    uint32_t *error_word;/* [1] sticky FC_ERR_* bits                             */
    /* per-request decode state (optional; NULL = every row in phase, none held) */
    int32_t *row_phase;  /* [B_cap] row b's decode step t_b = *step + row_phase[b]:
                            each request reranks at its own t_b % R == 0
                            (simulator.py:437-439, per-request r.t)          */
    uint8_t *row_hold;   /* [B_cap] FC_HOLD_* mode of row b for the next launches:
                            the reload pause of simulator.py:321-323,542     */
    uint64_t *stats;     /* [FC_STATS_N] device counters (Metrics,
                            simulator.py:87-131), or NULL                    */
} fc_store;

/* row_hold modes (the reloading request pauses; the others decode) */
#define FC_HOLD_NONE    0   /* decode normally                                   */
#define FC_HOLD_RERANK  3   /* rerank step of a two-tier row whose promoted pages
                               arrive on a side stream: score / select / recycle,
                               but no attention and no advance (t_b stays)       */
#define FC_HOLD_WAIT    1   /* reload in flight: nothing runs for the row        */
#define FC_HOLD_RESUME  2   /* reload landed: attend token t_b over the selection
                               made at the rerank step (stable heads not re-due) */

/* stats counters (each += per step by the kernels that do the work) */
#define FC_STAT_SCORE_EVALS        0  /* heads scored (Metrics.score_evals)        */
#define FC_STAT_SCORE_EVALS_NAIVE  1  /* L*H per decoding row (score_evals_naive)  */
#define FC_STAT_LAYER_SKIPS        2  /* (row, layer) with no due head
                                         (layer_scoring_skips)                     */
#define FC_STAT_HELD_ROW_STEPS     3  /* rows held for a reload (pause_steps)      */
#define FC_STATS_N                 4

/* library identity */
const char *fc_version(void);
/* last CUDA error string seen by this thread (for FC_E_CUDA) */
const char *fc_last_error(void);

/* ---- (4) allocation and step bookkeeping ------------------------------- */

/* Release every page of request row `row` (all layers, all heads) to the
 * free list, empty its selections and mark it free (seq_len = -1; a free row
 * is skipped by every kernel, fc_step_advance included): a finished request
 * in the serving loop.  Free-list order is not deterministic. */
int fc_free_row(const fc_store *s, int row, void *stream);

/* Allocate logical pages [first_page, first_page+n_pages) for every
 * (layer, head) of request row `row`, popping the device free list in
 * (layer, head, page) order — the order of the reference prefill, which
 * calls BlockTable.allocate_pages per head (simulator.py:361-364,
 * blocktable.py:236-246, PhysicalPool.allocate_many :59-71). */
int fc_alloc_pages(const fc_store *s, int row, int first_page, int n_pages,
                   void *stream);

/* End of a decode step for rows [0, batch): seq_len += 1; rows whose new
 * length starts a page get that page for every (layer, head), popped in
 * (row, layer, head) order — BlockTable.allocate_page_all_heads
 * (blocktable.py:248-263) as driven by simulator._append_token
 * (simulator.py:455-466) — and the page joins every head's current
 * selection (n_sel > 0): the page being written is always attended, as
 * the simulator's "resident ∪ appended" (simulator.py:463-466,512), so a
 * selection row is always the complete attended set.  Advances *step. */
int fc_step_advance(const fc_store *s, int batch, void *stream);

/* fc_step_advance that also counts, into s->stats (when set), the step's
 * layers with no due head per decoding row (Metrics.layer_scoring_skips,
 * simulator.py:440-446; `unstable` [L][H] flags, rerank period R).  Both
 * forms honour s->row_phase / s->row_hold: a held row keeps its length and
 * its own step t_b (simulator.py:321-323 — a paused request does not step). */
int fc_step_advance_counted(const fc_store *s, int batch, const uint8_t *unstable, int period,
                            void *stream);

/* ---- (1) KV append + per-page min/max summaries ------------------------ */

/* Prefill: write tokens [0, n_tokens) of request `row`, layer `layer` for
 * all H heads from k/v [H][n_tokens][d] (store dtype) into their pages and
 * build the page summaries — build_minmax (scoring.py:72-90). */
int fc_kv_prefill(const fc_store *s, int row, int layer, const void *k,
                  const void *v, int n_tokens, void *stream);

/* Decode append for rows [0, batch) of layer `layer`: write k_new/v_new
 * [batch][H][d] at position seq_len[row] and fold the key into that page's
 * summary — update_minmax (scoring.py:59-69).  Does not advance seq_len. */
int fc_kv_append(const fc_store *s, int layer, const void *k_new,
                 const void *v_new, int batch, void *stream);

/* Read back logical K/V of one (row, layer, head): pages [0, n_pages) into
 * k_out/v_out [n_pages*ps][d] (store dtype), undoing the in-page swizzle.
 * Non-resident pages are written as zeros. Test/offload helper. */
int fc_kv_gather(const fc_store *s, int row, int layer, int head, int n_pages,
                 void *k_out, void *v_out, void *stream);

/* ---- (2) page scoring + top-K selection -------------------------------- */

/* For every due (row, head) of `layer` among rows [0, batch): score its
 * pages with the GQA group bound (Quest; score_pages scoring.py:102-111,
 * summed over the G query heads) and select the top `topk` pages with the
 * last page pinned (select_topk scoring.py:164-193) into sel/n_sel.
 * Due = unstable[layer*H+h] || force_due || (*step % period == 0)
 * (rerank_due scoring.py:196-202).  `extra_tokens` (0 or 1) is added to
 * seq_len to count the token being appended this step.
 * q: [batch][H*G][d] (store dtype).  scores_out: [B_cap*H][pages_cap] fp32
 * workspace that receives the scores (pinned page = -inf).  counters:
 * [B_cap*H] int32, zero-initialised once by the caller.  kv_prefetch = 1:
 * the previous launch on the stream does not write this layer's summaries,
 * selections or seq_len, so the launch plans its range and warms L2 before
 * waiting for it (programmatic dependent launch); only q is waited for. */
size_t fc_score_select_workspace_size(const fc_store *s);
int fc_score_select(const fc_store *s, int layer, const void *q,
                    const uint8_t *unstable, int period, int force_due,
                    int topk, int extra_tokens, int kv_prefetch, float *scores_out,
                    int32_t *counters, int batch, void *stream);

/* Score only (no selection): scores_out[(row*H+h)*pages_cap + p] for pages
 * [0, n_pages) of every (row, head) of `layer` — score_pages. Used by the
 * per-head API and the parity tests. */
int fc_score_pages(const fc_store *s, int layer, const void *q,
                   int extra_tokens, float *scores_out, int batch,
                   void *stream);

/* Select only: top-K over caller-provided scores [n_heads][stride] fp32
 * with n_valid[i] candidates, pinning page n_valid[i]-1 when pin_last != 0.
 * Output sel_out [n_heads][topk] ascending, n_out [n_heads].
 * select_topk (scoring.py:164-193) bit-for-bit on the given scores. */
int fc_select_topk(const float *scores, int stride, const int32_t *n_valid,
                   int n_heads, int topk, int pin_last, int32_t *sel_out,
                   int32_t *n_out, void *stream);

/* select_topk (scoring.py:164-193) exactly on float64 scores[n] (the
 * reference's own precision, no rounding to fp32 keys): the min(k, n)
 * pages with the highest scores, ties to the lower index, pin_last: page
 * n-1 always in; sel_out[k] ascending, *n_out the count.  workspace: n
 * bytes.  n <= 12288. */
int fc_select_topk_f64(const double *scores, int n, int topk, int pin_last,
                       uint8_t *workspace, int32_t *sel_out, int32_t *n_out,
                       void *stream);

/* ---- (3) paged sparse decode attention ---------------------------------- */

/* For every (row, head) of `layer` among rows [0, batch): attend its query
 * group q[row][h*G .. h*G+G) to the tokens of the pages
 *   sel[0..n_sel) ∪ (max(sel), n_pages)           (n_sel == 0: all pages)
 * — sparse_decode / dense_decode (attention.py:76-111) with the stable-head
 * rule "selection at the last rerank plus pages appended since"
 * (simulator.py:416-420,512).  attend_appended = 0 attends exactly
 * sel[0..n_sel) (the per-call reference sparse_decode contract).
 * softmax scale = scale (1/sqrt(d) in the reference, attention.py:69).
 * Fused append: when k_new/v_new ([batch][H][d], store dtype) are given
 * (decode, extra_tokens = 1), the CTA that stages a head's last page writes
 * the new token into it and folds the key into the page summary
 * (update_minmax, scoring.py:59-69) — fc_kv_append in the same launch.
 * out: [batch][H*G][d] store dtype; lse: optional [batch][H*G] fp32
 * natural-log sum-exp.  Each head is processed by a cluster of S CTAs
 * (n_ctas = S; 0 = auto: the largest power of two <= 16 keeping all heads in
 * one wave); the CTAs of a cluster merge their softmax states through
 * distributed shared memory.  `max_pages` bounds the attended pages of any
 * head.  The workspace is a small scratch kept for ABI stability.
 * kv_prefetch = 1 lets the launch resolve pages and start their loads before
 * the previous kernel on the stream completes (programmatic dependent
 * launch); only q and k_new/v_new are waited for.  Valid when no kernel
 * between this layer's last selection/table update and this call is still
 * writing them (e.g. layers without a scoring launch this step).
 * early_unstable (optional, [layers][H] u8) with early_period: heads that
 * the preceding fc_score_select of this layer does not select this step
 * (not unstable and step % early_period != 0 — the same rerank_due rule)
 * start without waiting for it, overlapping the scoring of the due heads;
 * due heads wait as usual.  Pass null when a kernel other than that
 * fc_score_select (e.g. fc_rerank_recycle) precedes the call. */
size_t fc_sparse_decode_workspace_size(const fc_store *s, int batch,
                                       int max_pages, int n_ctas);
int fc_sparse_decode(const fc_store *s, int layer, const void *q,
                     const void *k_new, const void *v_new, void *out,
                     float *lse, float scale, int extra_tokens,
                     int attend_appended, int kv_prefetch,
                     const uint8_t *early_unstable, int early_period,
                     int max_pages, int n_ctas,
                     void *workspace, size_t ws_bytes, int batch,
                     void *stream);

/* fc_score_select followed by fc_sparse_decode of the same layer, fused:
 * per (row, head) one CTA — or, for small batches, a cluster of CTAs whose
 * keys meet in rank 0's shared memory — scores and selects (as
 * fc_score_select: score_pages / select_topk / rerank_due, scoring.py:93-202)
 * and then attends over the selection it just wrote (as fc_sparse_decode:
 * sparse_decode, attention.py:85-111, fused update_minmax, scoring.py:59-69).
 * Same results as the two calls; no grid-wide wait between them.
 * fc_score_attend_supported returns the CTAs per head it uses for this batch,
 * 0 when the geometry does not fit (FC_E_UNSUPPORTED: the caller issues the
 * two calls). */
int fc_score_attend_supported(const fc_store *s, int batch);
int fc_score_attend(const fc_store *s, int layer, const void *q,
                    const uint8_t *unstable, int period, int force_due,
                    int topk, int extra_tokens, int kv_prefetch,
                    float *scores_out, const void *k_new, const void *v_new,
                    void *out, float *lse, float scale, int attend_appended,
                    int batch, void *stream);
/* fc_score_attend over an explicit CTA map (mixed clusters): n_ctas CTAs in
 * clusters of `cluster` (2..16); cta_map [n_ctas] int32 gives each CTA its
 * (row * kv_heads + head): the `cluster` CTAs of a cluster that all name the
 * same head split it as fc_score_attend's clusters do; an entry with bit 30
 * set attends that head alone (scoring and selecting it too when it is due);
 * -1 leaves the CTA idle.  Every (row, head) in [0, batch * kv_heads) must
 * appear exactly once (a split cluster counts once).  Results are identical
 * to fc_score_attend for any such map; the map only balances the work — e.g.
 * the heads scored this step get a cluster each and the others share
 * clusters one per CTA, or every head is split and the scored ones are
 * listed first (clusters start in map order; a grid larger than one wave
 * runs in waves — clusters never wait on each other).
 * fc_score_attend_map_fits: 1 when a cluster of `cluster` CTAs of this
 * kernel fits on the device (n_ctas a multiple of it). */
int fc_score_attend_map_fits(const fc_store *s, int n_ctas, int cluster);
/* fc_score_attend with the scoring balanced over the whole GPU: one wave of
 * max(batch * kv_heads, SMs) co-resident CTAs first scores equal shares of
 * the concatenation of the due heads' candidate pages (as fc_score_select's
 * balanced kernel: the same per-page scores), then CTA i selects head i when
 * it is due (after every share of its scores landed; select_topk with the
 * last page pinned, scoring.py:164-193) and attends head i (sparse_decode,
 * attention.py:85-111, with the fused update_minmax).  For layers where only
 * some heads are due the summaries then stream at the GPU's rate rather than
 * one SM's.  counters: [batch_cap * kv_heads] int32, zero, left zero.
 * bf16 only; fc_score_attend_balanced_supported returns the grid it uses for
 * this batch, 0 when it does not fit (FC_E_UNSUPPORTED). */
int fc_score_attend_balanced_supported(const fc_store *s, int batch);
int fc_score_attend_balanced(const fc_store *s, int layer, const void *q,
                             const uint8_t *unstable, int period, int force_due,
                             int topk, int extra_tokens, int kv_prefetch,
                             float *scores_out, int32_t *counters,
                             const void *k_new, const void *v_new, void *out,
                             float *lse, float scale, int attend_appended,
                             int batch, void *stream);
/* fc_score_attend_balanced with the scored heads' attention cut into chunks
 * (FC_BAL_CHUNKS, 2..4, default 4) that the owner CTA and every CTA with no
 * work left claim; the CTA finishing a head's last chunk merges the chunk
 * states (same results up to the order of the softmax merge).  helper_ws:
 * fc_score_attend_balanced_workspace_size bytes, zero before the first call
 * and then kept for every later call of the same batch size (per-head words
 * and a launch epoch the kernel advances itself); NULL = no chunking. */
size_t fc_score_attend_balanced_workspace_size(const fc_store *s, int batch);
int fc_score_attend_balanced_ws(const fc_store *s, int layer, const void *q,
                                const uint8_t *unstable, int period, int force_due,
                                int topk, int extra_tokens, int kv_prefetch,
                                float *scores_out, int32_t *counters,
                                const void *k_new, const void *v_new, void *out,
                                float *lse, float scale, int attend_appended,
                                int batch, void *helper_ws, size_t helper_ws_bytes,
                                void *stream);
int fc_score_attend_map(const fc_store *s, int layer, const void *q,
                        const uint8_t *unstable, int period, int force_due,
                        int topk, int extra_tokens, int kv_prefetch,
                        float *scores_out, const void *k_new,
                        const void *v_new, void *out, float *lse, float scale,
                        int attend_appended, int batch, const int32_t *cta_map,
                        int n_ctas, int cluster, void *stream);

/* Persistent form of fc_sparse_decode for a run of consecutive layers
 * [layer_begin, layer_begin + n_layers) in ONE launch (same semantics per
 * (layer, head) as fc_sparse_decode: sparse_decode, attention.py:85-111, the
 * attended set of simulator.py:416-420,512, fused update_minmax,
 * scoring.py:59-69).  Where every head's cluster of CTAs can be co-resident
 * the kernel is the per-layer one's decomposition (one head per cluster,
 * fc_sparse_decode_layers_split) looping over the layers; otherwise one CTA
 * per SM with every layer's attended pages cut into equal ranges over all
 * warps of the grid.  A grid barrier separates layers (layer i's q and new
 * token are consumed only after every output of layer i-1 is written) while
 * page copies run ahead across it.  Layer
 * layer_begin + i reads q + i*q_layer_stride, k_new/v_new + i*kv_layer_stride
 * and writes out + i*out_layer_stride (elements), lse + i*lse_layer_stride
 * (optional).  No layer of the run may need a selection / table update
 * between layers (scoring, recycle): the host splits runs there.
 * first_dep = 1 when the previous launch on the stream writes layer
 * layer_begin's selection or table (its pages are then resolved after it
 * completes).  max_pages bounds the attended pages of any head.
 * Returns FC_E_UNSUPPORTED when the geometry does not fit (more than 256
 * heads per layer, or shared memory): callers use fc_sparse_decode.
 * workspace: fc_sparse_decode_layers_workspace_size() bytes, zeroed once
 * (its counters reset themselves). */
int fc_sparse_decode_layers_supported(const fc_store *s, int batch, int max_pages);
/* CTAs per head (cluster size) of the per-head persistent kernel that
 * fc_sparse_decode_layers uses for this batch, 0 when it falls back to the
 * warp-balanced persistent kernel. */
int fc_sparse_decode_layers_split(const fc_store *s, int batch, int max_pages);
size_t fc_sparse_decode_layers_workspace_size(const fc_store *s, int batch, int max_pages);
int fc_sparse_decode_layers(const fc_store *s, int layer_begin, int n_layers,
                            const void *q, int64_t q_layer_stride,
                            const void *k_new, const void *v_new, int64_t kv_layer_stride,
                            void *out, int64_t out_layer_stride,
                            float *lse, int64_t lse_layer_stride,
                            float scale, int extra_tokens, int attend_appended,
                            int first_dep, int max_pages,
                            void *workspace, size_t ws_bytes, int batch, void *stream);

/* ---- (4) stable-head rerank: recycle + tier copies ---------------------- */

/* For every stable (row, head) of `layer` due this step: diff the resident
 * set — old_sel[row][h][0..n_old) plus the pages appended since, i.e. every
 * page above max(old_sel) — against the new selection (store sel/n_sel),
 * pair evicted and promoted pages in ascending logical order and move their
 * blocks, release surplus / allocate deficit blocks, and emit the copy list
 * (row, head, logical page, dest block) — BlockTable.recycle
 * (blocktable.py:296-357), promoted_delta (tiering.py:42-46).
 * old_sel: [B_cap][H][sel_cap] int32, n_old: [B_cap][H] int32 (the
 * selection at the previous rerank; snapshot it before fc_score_select).
 * old_has_tail = 0 takes old_sel as the complete resident set (the per-call
 * reference recycle contract).  extra_tokens as in fc_score_select.
 * slow_resident: optional [B_cap][L][H][pages_cap] uint8, 1 = page has a
 * slow-tier copy (checked for every promoted page, blocktable.py:323-327).
 * copies: [max_copies][4] int32, n_copies: [1] int32 (appended atomically).
 * workspace: fc_rerank_workspace_size() bytes.  Unstable heads are skipped
 * (they never reload: tiering.py:164-166).  Within one call, surplus blocks
 * of all heads are pushed (head order, ascending pages) before deficits are
 * popped (head order, ascending pages); for a single head this is exactly
 * the reference order, across heads it matches up to block relabelling
 * (canonical_form, blocktable.py:414-428). */
size_t fc_rerank_workspace_size(const fc_store *s);
int fc_rerank_recycle(const fc_store *s, int layer, const int32_t *old_sel,
                      const int32_t *n_old, const uint8_t *unstable,
                      int period, int force_due, int old_has_tail,
                      int extra_tokens, const uint8_t *slow_resident,
                      int32_t *copies, int max_copies, int32_t *n_copies,
                      void *workspace, int batch, void *stream);
/* fc_rerank_recycle with an optional per-row mask row_skip [B_cap] uint8:
 * rows with row_skip[b] != 0 are treated as not due (no diff, no copies).
 * The serving loop sets it for requests whose post-prefill offload is still
 * in flight: they hold every page, so their resident set is not their old
 * selection (tiering.py:122-139 runs that offload in the background;
 * simulator.py:389-408 releases the pages only when it finishes).
 * row_skip = NULL is fc_rerank_recycle. */
int fc_rerank_recycle_rows(const fc_store *s, int layer, const int32_t *old_sel,
                           const int32_t *n_old, const uint8_t *unstable,
                           int period, int force_due, int old_has_tail,
                           int extra_tokens, const uint8_t *slow_resident,
                           const uint8_t *row_skip, int32_t *copies,
                           int max_copies, int32_t *n_copies,
                           void *workspace, int batch, void *stream);

/* Copy promoted pages from the pinned host slow tier into their HBM blocks:
 * copies [n][4] = (row, head, logical page, dest block) for layer `layer`;
 * host_pages is host-pinned memory [B_cap][L][H][N_cap][2][ps][d] (same
 * in-page layout as the pool), read with a zero-copy UVA gather kernel. */
/* fc_fetch_pages of the entries of request row `row` only (-1: every
 * entry) on at most max_ctas CTAs (0 = one per page up to 8 per SM): the
 * background fetch of a held row's promoted pages (reload pause) on a few
 * SMs beside the decode steps of the other rows, one launch per row so
 * each resumes as soon as its own pages landed. */
int fc_fetch_pages_ctas(const fc_store *s, int layer, const void *host_pages, const int32_t *copies,
                        const int32_t *n_copies, int max_copies, int row, int max_ctas, void *stream);
int fc_fetch_pages(const fc_store *s, int layer, const void *host_pages,
                   const int32_t *copies, const int32_t *n_copies,
                   int max_copies, void *stream);

/* Reload staging — the paper's transfer/compute overlap:
 * fc_stage_promoted diffs a PREDICTED selection (pred_sel / pred_n, same
 * layout as the store's sel / n_sel, e.g. fc_score_select into a second
 * fc_store view some steps before a rerank) of every stable (row, layer,
 * head) against its resident set (its current selection) and fetches the
 * pages it would promote that have a slow-tier copy (slow_resident) from
 * host_pages into `staging` ([capacity] pages of device memory), recording
 * staged_map[row][layer][head][page] = slot (-1 elsewhere) and stage_list
 * [capacity][2] = (flat head, page); *stage_count counts them (pages past
 * capacity are simply not staged).  Run it on a side stream while decode
 * continues.  fc_fetch_pages_staged is fc_fetch_pages taking staged pages
 * from `staging` (HBM) instead of the host link (+1 on *n_staged_hits per
 * page, optional).  fc_stage_clear resets the map and the count after the
 * rerank.  The rerank (selection, BlockTable.recycle, copy list) is
 * unchanged: results are identical with or without staging. */
int fc_fetch_pages_staged(const fc_store *s, int layer, const void *host_pages,
                          const int32_t *copies, const int32_t *n_copies,
                          int max_copies, const int32_t *staged_map,
                          const void *staging, int32_t *n_staged_hits,
                          void *stream);
int fc_stage_promoted(const fc_store *s, const int32_t *pred_sel,
                      const int32_t *pred_n, const uint8_t *unstable,
                      const uint8_t *slow_resident, const void *host_pages,
                      int32_t *staged_map, int32_t *stage_list,
                      int32_t *stage_count, int capacity, void *staging,
                      int batch, void *stream);
/* The two halves of fc_stage_promoted: the diff / slot assignment (a few
 * microseconds) and the host -> staging copies (on a few SMs, for a side
 * stream beside decode).  Several predictions may stage before one rerank:
 * pass k (0..3) records its slot range in stage_count[1 + 2k .. 2 + 2k]
 * (stage_count has 9 ints; fc_stage_promoted is pass 0) and fc_stage_fetch
 * of pass k copies exactly that range. */
int fc_stage_plan(const fc_store *s, const int32_t *pred_sel,
                  const int32_t *pred_n, const uint8_t *unstable,
                  const uint8_t *slow_resident, int32_t *staged_map,
                  int32_t *stage_list, int32_t *stage_count, int capacity,
                  int batch, int pass, void *stream);
int fc_stage_fetch(const fc_store *s, const void *host_pages,
                   const int32_t *stage_list, const int32_t *stage_count,
                   int capacity, void *staging, int pass, void *stream);
int fc_stage_clear(const fc_store *s, int32_t *staged_map,
                   const int32_t *stage_list, int32_t *stage_count,
                   int capacity, void *stream);

/* Offload full pages of stable heads to the pinned host slow tier:
 * pages [n][4] = (row, layer, head, logical page), one write per page
 * (TierStore._record write-once ledger, tiering.py:99-157). */
int fc_offload_pages(const fc_store *s, void *host_pages, const int32_t *pages,
                     int n_pages, void *stream);
/* fc_offload_pages on at most max_ctas CTAs (0 = as many as fill the GPU):
 * a background offload that leaves the other SMs to decode steps running
 * concurrently on another stream (the post-prefill offload in serving). */
int fc_offload_pages_ctas(const fc_store *s, void *host_pages, const int32_t *pages,
                          int n_pages, int max_ctas, void *stream);

/* Per-step incremental offload of stable heads (tiering.py:141-157, driven
 * as simulator._append_token, simulator.py:467-477): for rows [0, batch)
 * whose seq_len is a positive multiple of ps (the page seq_len/ps - 1 just
 * filled), copy that page of every stable (layer, head) to the pinned host
 * tier and set slow_resident[row][l][h][page]; a page already marked sets
 * FC_ERR_WRITE_TWICE (write-once ledger).  Run after fc_step_advance. */
int fc_offload_filled(const fc_store *s, void *host_pages, const uint8_t *unstable,
                      uint8_t *slow_resident, int batch, void *stream);

/* After the post-prefill offload: release every page of every stable head of
 * rows [0, batch) that is not in its current selection (the offload_done
 * eviction, simulator.py:389-408).  Blocks return to the free list in an
 * unspecified order (naming is canonical-equivalent). */
int fc_evict_unselected(const fc_store *s, const uint8_t *unstable, int batch,
                        void *stream);

/* Evict (set to the null block and release) logical pages listed in
 * pages [n][4] = (row, layer, head, logical page) — evict_many
 * (blocktable.py:280-294). */
int fc_evict_pages(const fc_store *s, const int32_t *pages, int n_pages,
                   void *stream);

/* ---- (f2) selection traces and head stability --------- */

/* Copy the current top-K selection of every (row < batch, layer, head) into
 * trace slot (*step - step_base) of a device trace buffer, skipped when the
 * slot is outside [0, n_slots):
 *   trace_sel  [batch_cap][n_slots][L][H][topk] u32 — FXTK records, layer-
 *              major, head-minor (trace.py:1-19);
 *   trace_pool [batch_cap][n_slots] u32 — candidate pool size,
 *              ceil((seq_len + extra_tokens) / ps).
 * Run after the step's scoring with every head due (a profiling step); a
 * selection shorter than topk (pool <= K) sets FC_ERR_TRACE_SHORT and writes
 * 0xffffffff.  Graph-capturable (the slot comes from the device step). */
int fc_trace_capture(const fc_store *s, uint32_t *trace_sel, uint32_t *trace_pool,
                     int step_base, int n_slots, int topk, int extra_tokens,
                     int batch, void *stream);

/* Integer core of the random-corrected overlap (stability.py:24-62) over a
 * device trace sel [n_steps][L][H][topk] u32, pool [n_steps] u32:
 * inter[l][h][w][delta-1] = |sel[starts[w]] ∩ sel[starts[w]+delta]| for
 * delta in 1..window-1, or -1 when pool[starts[w]+delta] <= topk
 * (degenerate pair).  starts: device int32 [n_windows], each with
 * starts[w] + window - 1 < n_steps (checked by the caller); max_pool bounds
 * every page index + 1 (indices at or above it never match). */
int fc_trace_overlap(const uint32_t *sel, const uint32_t *pool, int n_steps,
                     int layers, int kv_heads, int topk, const int32_t *starts,
                     int n_windows, int window, int max_pool, int32_t *inter,
                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLEXICACHE_B200_H */
