// recycle.cu — subsystem (4): stable-head rerank block recycling and the
// pinned-host slow tier copies.
//
// Reference semantics:
//   BlockTable.recycle  blocktable.py:296-357  evicted = old\new, promoted =
//       new\old, paired ascending; surplus evictions freed, deficit allocated;
//       copy list (promoted page, dest block); validations :313-327
//   promoted_delta      tiering.py:42-46
//   TierStore offload / reload (write-once ledger)  tiering.py:99-173
//   simulator._rerank   simulator.py:500-547 (base = resident ∪ appended)
//
// The rerank is two launches per layer at a rerank step: a warp per head
// computes the ascending diff with ballots and moves paired blocks in place
// (the paper's fused recycle kernel), then one CTA applies
// the free-list pushes/pops for all heads in head order.  Copies between the
// pinned host tier and HBM are zero-copy UVA kernels: a
// CTA per page moves 8 KiB with 16-byte loads, so many PCIe reads are in
// flight without one cudaMemcpy per page.
#include "store.cuh"
#include <cub/block/block_scan.cuh>

namespace fc {

constexpr int kRecycleWarps = 4;
constexpr int kListCap = 1024;  // max entries of an old/new selection list
constexpr int kRecycleSlack = 64;  // pages appended since the old selection (old_has_tail)

// per head bh: [4 counts: surplus, deficit, pairs m, -][evicted pages][their
// blocks][promoted pages], kListCap each, ascending.  The first m evicted /
// promoted entries are the pairs; the surplus blocks and deficit pages follow.
// The commit kernel reads the whole diff, so when the pool cannot cover the
// deficits it puts every paired move back before anything else changes
// (BlockTable.recycle validates before mutating, blocktable.py:313-331).
constexpr int kWsPerHead = 4 + 3 * kListCap;
struct RerankWs {
    int32_t *base;
    __device__ __forceinline__ int32_t *cnt(int bh) const { return base + (int64_t)bh * kWsPerHead; }
    __device__ __forceinline__ int32_t *ev_page(int bh) const { return cnt(bh) + 4; }
    __device__ __forceinline__ int32_t *ev_blk(int bh) const { return cnt(bh) + 4 + kListCap; }
    __device__ __forceinline__ int32_t *pr_page(int bh) const { return cnt(bh) + 4 + 2 * kListCap; }
    __device__ __forceinline__ int32_t *freed(int bh) const { return ev_blk(bh) + cnt(bh)[2]; }
    __device__ __forceinline__ int32_t *alloc(int bh) const { return pr_page(bh) + cnt(bh)[2]; }
};

FC_DEVINL bool sorted_contains(const int32_t *a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == x;
}

// The diff of one head by one warp (every lane calls it).  w_smem: the
// warp's old list | new list | old blocks | evicted | evicted blocks |
// promoted, sel_cap + slack entries each (both selections are staged in
// shared memory first: the membership tests are binary searches, which
// through global memory would chain ~8 dependent loads per entry).
FC_DEVINL void rerank_diff_head(const StoreView &s, int layer, const int32_t *__restrict__ old_sel,
                                const int32_t *__restrict__ n_old_arr, const uint8_t *__restrict__ unstable,
                                int period, int force_due, int old_has_tail, int extra_tokens,
                                const uint8_t *__restrict__ slow_resident, const uint8_t *__restrict__ row_skip,
                                int32_t *copies, int max_copies, int32_t *n_copies, RerankWs ws, int bh,
                                int32_t *w_smem) {
    const int lane = threadIdx.x & 31;
    const int cap = s.SELCAP + kRecycleSlack;  // old list incl. pages appended since (old_has_tail)
    int32_t *s_old = w_smem;
    int32_t *s_new = s_old + cap;
    int32_t *s_oblk = s_new + cap;   // block of old entry i
    int32_t *s_evw = s_oblk + cap;   // evicted pages, ascending
    int32_t *s_evblk = s_evw + cap;  // their blocks
    int32_t *s_prw = s_evblk + cap;  // promoted pages, ascending
    const int b = bh / s.H, h = bh % s.H;
    int32_t *cnt = ws.cnt(bh);
    // rows in row_skip still hold every page (post-prefill offload in flight):
    // their resident set is not the old selection, so nothing moves
    const bool due = !unstable[layer * s.H + h] && (force_due || s.boundary(*s.step, b, period)) &&
                     !(row_skip && row_skip[b]);
    if (!due) {
        if (lane == 0) { cnt[0] = 0; cnt[1] = 0; cnt[2] = 0; }
        return;
    }
    const int hx = s.hix(b, layer, h);
    const int n_pages = (s.seq_len[b] + extra_tokens + s.PS - 1) / s.PS;
    const int32_t *olds = old_sel + (int64_t)bh * s.SELCAP;
    const int n_old_sel = n_old_arr[bh];
    const int hi_old = n_old_sel > 0 ? olds[n_old_sel - 1] : -1;
    // resident set = old selection + pages appended since (simulator.py:512)
    const int n_old = old_has_tail ? n_old_sel + max(0, n_pages - 1 - hi_old) : n_old_sel;
    const int hi_res = old_has_tail ? max(hi_old, n_pages - 1) : hi_old;
    const int32_t *news = s.sel + (int64_t)hx * s.SELCAP;
    const int n_new = s.n_sel[hx];
    int32_t *trow = s.table + s.table_off(hx, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (n_old_sel > s.SELCAP || n_new > s.SELCAP) {
        if (lane == 0) { set_error(s.err, FC_ERR_SEL_CAP); cnt[0] = 0; cnt[1] = 0; cnt[2] = 0; }
        return;
    }
    for (int i = lane; i < n_old_sel; i += 32) s_old[i] = olds[i];
    for (int i = lane; i < n_new; i += 32) s_new[i] = news[i];
    __syncwarp();

    // blocks of the old entries: every lane's loads issued before any use
    // (this validation was a chain of dependent table reads per 32 entries)
    if (n_old > cap) {
        if (lane == 0) { set_error(s.err, FC_ERR_SEL_CAP); cnt[0] = 0; cnt[1] = 0; cnt[2] = 0; }
        return;
    }
    for (int base = 0; base < n_old; base += 128) {
        int xs[4], bl[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = base + u * 32 + lane;
            xs[u] = i < n_old ? (i < n_old_sel ? s_old[i] : hi_old + 1 + (i - n_old_sel)) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) bl[u] = xs[u] >= 0 ? trow[xs[u]] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (xs[u] < 0) continue;
            s_oblk[base + u * 32 + lane] = bl[u];
            if (bl[u] == FC_NULL_BLOCK) set_error(s.err, FC_ERR_DOUBLE_EVICT);
        }
    }
    __syncwarp();
    // evicted = old \ new (ascending)
    int n_ev = 0;
    for (int base = 0; base < n_old; base += 32) {
        const int i = base + lane;
        bool ev = false;
        int x = 0;
        if (i < n_old) {
            x = i < n_old_sel ? s_old[i] : hi_old + 1 + (i - n_old_sel);
            ev = !sorted_contains(s_new, n_new, x);
        }
        const unsigned mk = __ballot_sync(0xffffffffu, ev);
        if (ev) {
            const int r = n_ev + __popc(mk & lt);
            if (r < cap) { s_evw[r] = x; s_evblk[r] = s_oblk[i]; }
        }
        n_ev += __popc(mk);
    }
    // promoted = new \ old (ascending), then their validations (non-resident,
    // slow copy present) with every lane's loads in flight together
    int n_pr = 0;
    for (int base = 0; base < n_new; base += 32) {
        const int i = base + lane;
        bool pr = false;
        int x = 0;
        if (i < n_new) {
            x = s_new[i];
            pr = (x > hi_res) || (x <= hi_old && !sorted_contains(s_old, n_old_sel, x));
        }
        const unsigned mk = __ballot_sync(0xffffffffu, pr);
        if (pr) {
            const int r = n_pr + __popc(mk & lt);
            if (r < cap) s_prw[r] = x;
        }
        n_pr += __popc(mk);
    }
    __syncwarp();
    for (int base = 0; base < min(n_pr, cap); base += 128) {
        int bl[4], sr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = base + u * 32 + lane;
            const int x = i < min(n_pr, cap) ? s_prw[i] : -1;
            bl[u] = x >= 0 ? trow[x] : FC_NULL_BLOCK;
            sr[u] = (x >= 0 && slow_resident) ? slow_resident[s.table_off(hx, x)] : 1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (bl[u] != FC_NULL_BLOCK) set_error(s.err, FC_ERR_DOUBLE_EVICT);
            if (!sr[u]) set_error(s.err, FC_ERR_NULL_READ);
        }
    }
    if (n_ev > cap || n_pr > cap || n_ev > kListCap || n_pr > kListCap) {
        if (lane == 0) { set_error(s.err, FC_ERR_SEL_CAP); cnt[0] = 0; cnt[1] = 0; cnt[2] = 0; }
        return;
    }
    __syncwarp();
    const int m = min(n_ev, n_pr);
    int cbase = 0;
    if (lane == 0 && m > 0) cbase = atomicAdd(n_copies, m);
    cbase = __shfl_sync(0xffffffffu, cbase, 0);
    for (int i = lane; i < m; i += 32) {  // ascending pairs: evicted[i] hands its block to promoted[i]
        const int e = s_evw[i], p = s_prw[i];
        const int blk = s_evblk[i];
        trow[e] = FC_NULL_BLOCK;
        trow[p] = blk;
        if (cbase + i < max_copies) {
            int32_t *cp = copies + 4 * (int64_t)(cbase + i);
            cp[0] = b; cp[1] = h; cp[2] = p; cp[3] = blk;
        } else {
            set_error(s.err, FC_ERR_SEL_CAP);
        }
    }
    for (int i = m + lane; i < n_ev; i += 32) trow[s_evw[i]] = FC_NULL_BLOCK;  // surplus evictions
    // the whole diff for the commit (and its undo on pool exhaustion)
    int32_t *evp = ws.ev_page(bh), *evb = ws.ev_blk(bh), *prp = ws.pr_page(bh);
    for (int i = lane; i < n_ev; i += 32) { evp[i] = s_evw[i]; evb[i] = s_evblk[i]; }
    for (int i = lane; i < n_pr; i += 32) prp[i] = s_prw[i];
    if (lane == 0) { cnt[0] = n_ev - m; cnt[1] = n_pr - m; cnt[2] = m; }
}

__global__ void __launch_bounds__(kRecycleWarps * 32)
rerank_diff_kernel(StoreView s, int layer, const int32_t *__restrict__ old_sel,
                   const int32_t *__restrict__ n_old_arr, const uint8_t *__restrict__ unstable,
                   int period, int force_due, int old_has_tail, int extra_tokens,
                   const uint8_t *__restrict__ slow_resident, const uint8_t *__restrict__ row_skip,
                   int32_t *copies, int max_copies, int32_t *n_copies, RerankWs ws, int batch) {
    extern __shared__ int32_t dsm_r[];
    griddep_launch_dependents();
    griddep_wait();  // the selection comes from the scoring launch before
    const int w = threadIdx.x >> 5;
    const int bh = blockIdx.x * kRecycleWarps + w;
    if (bh >= batch * s.H) return;
    rerank_diff_head(s, layer, old_sel, n_old_arr, unstable, period, force_due, old_has_tail, extra_tokens,
                     slow_resident, row_skip, copies, max_copies, n_copies, ws, bh,
                     dsm_r + (int64_t)w * 6 * (s.SELCAP + kRecycleSlack));
}

// pushes of all heads (head order) then pops (head order); 1024 threads
FC_DEVINL void rerank_commit_body(const StoreView &s, int layer, int32_t *copies, int max_copies,
                                  int32_t *n_copies, RerankWs ws, int batch) {
    using Scan = cub::BlockScan<int, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int s_fail;
    const int nh = batch * s.H;
    const int top0 = *s.free_top;
    // pass 0: can the pool cover every deficit (after the surplus pushes)?
    // If not, undo the diff kernel's moves, emit no copies and leave the free
    // list untouched: PoolExhausted with the table as before (blocktable.py:59-71)
    {
        int net = 0;
        for (int bh = threadIdx.x; bh < nh; bh += 1024) net += ws.cnt(bh)[1] - ws.cnt(bh)[0];
        int before, total;
        Scan(tmp).ExclusiveSum(net, before, total);
        __syncthreads();
        if (top0 - total < 0) {
            for (int bh = threadIdx.x; bh < nh; bh += 1024) {
                const int *c = ws.cnt(bh);
                const int m = c[2], n_ev = m + c[0];
                if (n_ev == 0 && m == 0) continue;
                const int b = bh / s.H, h = bh % s.H;
                int32_t *trow = s.table + s.table_off(s.hix(b, layer, h), 0);
                for (int i = 0; i < m; ++i) trow[ws.pr_page(bh)[i]] = FC_NULL_BLOCK;
                for (int i = 0; i < n_ev; ++i) trow[ws.ev_page(bh)[i]] = ws.ev_blk(bh)[i];
            }
            if (threadIdx.x == 0) { *n_copies = 0; set_error(s.err, FC_ERR_POOL_EXHAUSTED); }
            return;
        }
    }
    // pass 1: pushes
    int fcarry = 0;
    for (int c0 = 0; c0 < nh; c0 += 1024) {
        const int bh = c0 + threadIdx.x;
        const int f = bh < nh ? ws.cnt(bh)[0] : 0;
        int before, total;
        Scan(tmp).ExclusiveSum(f, before, total);
        for (int k = 0; k < f; ++k) s.free_stack[top0 + fcarry + before + k] = ws.freed(bh)[k];
        fcarry += total;
        __syncthreads();
    }
    const int top1 = top0 + fcarry;
    // pass 2: pops
    int acarry = 0;
    for (int c0 = 0; c0 < nh; c0 += 1024) {
        const int bh = c0 + threadIdx.x;
        const int a = bh < nh ? ws.cnt(bh)[1] : 0;
        int before, total;
        Scan(tmp).ExclusiveSum(a, before, total);
        if (threadIdx.x == 0) s_fail = (top1 - acarry - total < 0);
        __syncthreads();
        if (!s_fail && a > 0) {
            const int b = bh / s.H, h = bh % s.H;
            const int hx = s.hix(b, layer, h);
            const int cb = atomicAdd(n_copies, a);
            for (int k = 0; k < a; ++k) {
                const int page = ws.alloc(bh)[k];
                const int blk = s.free_stack[top1 - 1 - (acarry + before + k)];
                s.table[s.table_off(hx, page)] = blk;
                if (cb + k < max_copies) {
                    int32_t *cp = copies + 4 * (int64_t)(cb + k);
                    cp[0] = b; cp[1] = h; cp[2] = page; cp[3] = blk;
                } else {
                    set_error(s.err, FC_ERR_SEL_CAP);
                }
            }
        }
        if (s_fail) {
            if (threadIdx.x == 0) set_error(s.err, FC_ERR_POOL_EXHAUSTED);
            break;
        }
        acarry += total;
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) *s.free_top = top1 - acarry;
}

__global__ void __launch_bounds__(1024)
rerank_commit_kernel(StoreView s, int layer, int32_t *copies, int max_copies, int32_t *n_copies,
                     RerankWs ws, int batch) {
    griddep_launch_dependents();
    griddep_wait();
    rerank_commit_body(s, layer, copies, max_copies, n_copies, ws, batch);
}

// Few heads (<= 32, e.g. one request): the diffs (warp w: head w) and the
// commit in ONE CTA — one launch and one dependency hand-off per layer
// instead of two.  Same results as the two kernels.
__global__ void __launch_bounds__(1024)
rerank_small_kernel(StoreView s, int layer, const int32_t *__restrict__ old_sel,
                    const int32_t *__restrict__ n_old_arr, const uint8_t *__restrict__ unstable,
                    int period, int force_due, int old_has_tail, int extra_tokens,
                    const uint8_t *__restrict__ slow_resident, const uint8_t *__restrict__ row_skip,
                    int32_t *copies, int max_copies, int32_t *n_copies, RerankWs ws, int batch) {
    extern __shared__ int32_t dsm_r[];
    griddep_launch_dependents();
    griddep_wait();  // the selection comes from the scoring launch before
    const int w = threadIdx.x >> 5;
    if (w < batch * s.H)
        rerank_diff_head(s, layer, old_sel, n_old_arr, unstable, period, force_due, old_has_tail, extra_tokens,
                         slow_resident, row_skip, copies, max_copies, n_copies, ws, w,
                         dsm_r + (int64_t)w * 6 * (s.SELCAP + kRecycleSlack));
    __syncthreads();  // every head's diff (global workspace, table) before the commit
    rerank_commit_body(s, layer, copies, max_copies, n_copies, ws, batch);
}

// ---------------------------------------------------------------------------
// pinned-host <-> HBM page copies (zero-copy UVA)

constexpr int kCopyThreads = 128;

FC_DEVINL void copy_page(uint4 *dst, const uint4 *src, int n16) {
    constexpr int U = 4;
    for (int i0 = threadIdx.x; i0 < n16; i0 += kCopyThreads * U) {
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kCopyThreads;
            if (i < n16) r[u] = src[i];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = i0 + u * kCopyThreads;
            if (i < n16) dst[i] = r[u];
        }
    }
}

// staged_map (optional, [B][L][H][NCAP] int32, -1 = not staged): a promoted
// page staged ahead of the rerank (stage_fetch_kernel) is copied from the
// staging area in HBM instead of over the host link.
//
// CTAs of 128 threads, 16-byte register loads, 4 in flight per thread: 51
// GB/s for random 8 KiB pages from 32 CTAs up (55 GB/s for a
// cudaMemcpy of one contiguous buffer; scripts/micro/fetch_bw.cu).  The CTAs
// need no shared memory, so they run beside the decode kernels, which hold
// ~200 KB of it per SM (a bulk-copy variant through shared memory reached
// the same 51 GB/s alone but could only start between decode launches: 0.92
// of the rows' steps held at config 3); capping the grid keeps the SMs they
// take few (PAPER.md: "capping grid size to keep SM occupancy low").
__global__ void __launch_bounds__(kCopyThreads)
fetch_kernel(StoreView s, int layer, const char *host_pages, const int32_t *copies,
             const int32_t *n_copies, int max_copies, int page_bytes, const int32_t *staged_map,
             const char *staging, int32_t *n_staged_hits, int row) {
    griddep_launch_dependents();
    griddep_wait();  // the copy list comes from the recycle launch before
    const int n = min(*n_copies, max_copies);
    for (int c = blockIdx.x; c < n; c += gridDim.x) {
        const int b = copies[4 * c], h = copies[4 * c + 1], p = copies[4 * c + 2], blk = copies[4 * c + 3];
        if (row >= 0 && b != row) continue;  // (one request's pages: it resumes when they landed)
        const int64_t off = s.table_off(s.hix(b, layer, h), p);
        const int slot = staged_map ? staged_map[off] : -1;
        const char *src = slot >= 0 ? staging + (int64_t)slot * page_bytes : host_pages + off * (int64_t)page_bytes;
        if (slot >= 0 && threadIdx.x == 0 && n_staged_hits) atomicAdd(n_staged_hits, 1);
        copy_page(reinterpret_cast<uint4 *>(reinterpret_cast<char *>(s.pool) + (int64_t)blk * page_bytes),
                  reinterpret_cast<const uint4 *>(src), page_bytes / 16);
    }
}

// ---------------------------------------------------------------------------
// Reload staging (the paper's transfer/compute overlap, PAPER.md:221-224,
// realised for the request itself): a selection predicted some steps before
// a rerank (scored into a separate selection buffer) is diffed against the
// resident set (= the current selection of a stable head); pages it would
// promote that have a slow-tier copy are fetched host -> staging area on a
// side stream while decode continues.  At the rerank, fetch_kernel takes
// staged pages from HBM.  The rerank itself (selection, recycle, copy list)
// is unchanged, so results are identical with or without staging.

// one warp per (row, layer, head) of the stable heads
__global__ void __launch_bounds__(256)
stage_plan_kernel(StoreView s, const int32_t *pred_sel, const int32_t *pred_n, const uint8_t *unstable,
                  const uint8_t *slow_resident, int32_t *staged_map, int32_t *stage_list, int32_t *stage_count,
                  int cap, int batch) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int LH = s.L * s.H;
    if (warp >= batch * LH) return;
    const int b = warp / LH, lh = warp % LH, l = lh / s.H, h = lh % s.H;
    if (unstable[lh]) return;
    const int hx = s.hix(b, l, h);
    const int32_t *cur = s.sel + (int64_t)hx * s.SELCAP;
    const int ncur = s.n_sel[hx];
    const int32_t *pred = pred_sel + (int64_t)hx * s.SELCAP;
    const int npred = pred_n[hx];
    for (int i = lane; i < npred; i += 32) {
        const int p = pred[i];
        int lo = 0, hi = ncur;  // resident set = the current (ascending) selection
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cur[mid] < p) lo = mid + 1; else hi = mid;
        }
        if (lo < ncur && cur[lo] == p) continue;
        const int64_t off = s.table_off(hx, p);
        if (!slow_resident[off] || staged_map[off] >= 0) continue;
        const int slot = atomicAdd(stage_count, 1);
        if (slot >= cap) continue;  // staging area full: fetched from the host at the rerank
        staged_map[off] = slot;
        stage_list[2 * slot] = hx;
        stage_list[2 * slot + 1] = p;
    }
}

// stage_count layout: [0] slots taken; [1 + 2k], [2 + 2k] = first / end slot
// of staging pass k (several predictions may stage before one rerank)
constexpr int kStagePasses = 4;

__global__ void stage_mark_kernel(int32_t *stage_count, int idx) { stage_count[idx] = stage_count[0]; }

__global__ void __launch_bounds__(kCopyThreads)
stage_fetch_kernel(StoreView s, const char *host_pages, const int32_t *stage_list, const int32_t *stage_count,
                   int cap, char *staging, int page_bytes, int pass) {
    const int n = min(stage_count[2 + 2 * pass], cap);
    for (int c = min(stage_count[1 + 2 * pass], cap) + blockIdx.x; c < n; c += gridDim.x) {
        const int64_t off = s.table_off(stage_list[2 * c], stage_list[2 * c + 1]);
        copy_page(reinterpret_cast<uint4 *>(staging + (int64_t)c * page_bytes),
                  reinterpret_cast<const uint4 *>(host_pages + off * (int64_t)page_bytes), page_bytes / 16);
    }
}

__global__ void stage_clear_kernel(StoreView s, int32_t *staged_map, const int32_t *stage_list, int32_t *stage_count,
                                   int cap) {
    const int n = min(*stage_count, cap);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n; c += gridDim.x * blockDim.x)
        staged_map[s.table_off(stage_list[2 * c], stage_list[2 * c + 1])] = -1;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < 1 + 2 * kStagePasses && gridDim.x == 1) stage_count[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(kCopyThreads)
offload_kernel(StoreView s, char *host_pages, const int32_t *pages, int n, int page_bytes) {
    for (int c = blockIdx.x; c < n; c += gridDim.x) {
        const int b = pages[4 * c], l = pages[4 * c + 1], h = pages[4 * c + 2], p = pages[4 * c + 3];
        const int64_t off = s.table_off(s.hix(b, l, h), p);
        const int blk = s.table[off];
        if (blk == FC_NULL_BLOCK) {
            if (threadIdx.x == 0) set_error(s.err, FC_ERR_NULL_READ);
            continue;
        }
        copy_page(reinterpret_cast<uint4 *>(host_pages + off * page_bytes),
                  reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(s.pool) +
                                                  (int64_t)blk * page_bytes),
                  page_bytes / 16);
    }
}


// per-step incremental offload: grid-stride over (row, layer, head)
__global__ void __launch_bounds__(kCopyThreads)
offload_filled_kernel(StoreView s, char *host_pages, const uint8_t *unstable, uint8_t *slow_resident,
                      int batch, int page_bytes) {
    const int LH = s.L * s.H;
    for (int u = blockIdx.x; u < batch * LH; u += gridDim.x) {
        const int b = u / LH, lh = u % LH;
        if (unstable[lh]) continue;
        const int len = s.seq_len[b];
        if (len <= 0 || len % s.PS != 0 || !s.decodes(b)) continue;  // (a held row filled nothing)
        const int page = len / s.PS - 1;
        const int64_t off = s.table_off(s.hix(b, lh / s.H, lh % s.H), page);
        const int blk = s.table[off];
        if (blk == FC_NULL_BLOCK) {
            if (threadIdx.x == 0) set_error(s.err, FC_ERR_NULL_READ);
            continue;
        }
        if (slow_resident && slow_resident[off]) {
            if (threadIdx.x == 0) set_error(s.err, FC_ERR_WRITE_TWICE);
            continue;
        }
        copy_page(reinterpret_cast<uint4 *>(host_pages + off * page_bytes),
                  reinterpret_cast<const uint4 *>(reinterpret_cast<const char *>(s.pool) +
                                                  (int64_t)blk * page_bytes),
                  page_bytes / 16);
        __syncthreads();
        if (threadIdx.x == 0 && slow_resident) slow_resident[off] = 1;
    }
}

// release every non-selected page of stable heads: one CTA per (row, layer, head)
__global__ void __launch_bounds__(256)
evict_unselected_kernel(StoreView s, const uint8_t *unstable, int batch, int extra_tokens) {
    const int LH = s.L * s.H;
    const int u = blockIdx.x;
    if (u >= batch * LH) return;
    const int b = u / LH, lh = u % LH;
    if (unstable[lh]) return;
    const int hx = s.hix(b, lh / s.H, lh % s.H);
    const int n_pages = (s.seq_len[b] + extra_tokens + s.PS - 1) / s.PS;
    const int nsel = s.n_sel[hx];
    const int32_t *sel = s.sel + (int64_t)hx * s.SELCAP;
    int32_t *trow = s.table + s.table_off(hx, 0);
    for (int p = threadIdx.x; p < n_pages; p += blockDim.x) {
        // sel is ascending: binary search
        int lo = 0, hi = nsel;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sel[mid] < p) lo = mid + 1; else hi = mid;
        }
        if (lo < nsel && sel[lo] == p) continue;
        const int blk = trow[p];
        if (blk == FC_NULL_BLOCK) continue;
        trow[p] = FC_NULL_BLOCK;
        const int slot = atomicAdd(s.free_top, 1);
        s.free_stack[slot] = blk;
    }
}

// ---------------------------------------------------------------------------

size_t rerank_workspace_bytes(const StoreView &s) {
    return (size_t)s.B * s.H * kWsPerHead * sizeof(int32_t);
}

cudaError_t launch_rerank(const StoreView &s, int layer, const int32_t *old_sel, const int32_t *n_old,
                          const uint8_t *unstable, int period, int force_due, int old_has_tail,
                          int extra_tokens, const uint8_t *slow_resident, const uint8_t *row_skip,
                          int32_t *copies, int max_copies, int32_t *n_copies, void *workspace, int batch,
                          cudaStream_t st) {
    RerankWs ws{reinterpret_cast<int32_t *>(workspace)};
    const int heads = batch * s.H;
    const size_t smem1 = (size_t)heads * 6 * (s.SELCAP + kRecycleSlack) * sizeof(int32_t);
    if (heads <= 32 && smem1 <= 200 * 1024) {
        static size_t configured1 = 0;
        if (smem1 > 48 * 1024 && configured1 < smem1) {
            cudaError_t e = cudaFuncSetAttribute(rerank_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem1);
            if (e != cudaSuccess) return e;
            configured1 = smem1;
        }
        return launch_pdl(rerank_small_kernel, dim3(1), dim3(1024), smem1, st, s, layer, old_sel, n_old, unstable,
                          period, force_due, old_has_tail, extra_tokens, slow_resident, row_skip, copies, max_copies,
                          n_copies, ws, batch);
    }
    const size_t smem = (size_t)kRecycleWarps * 6 * (s.SELCAP + kRecycleSlack) * sizeof(int32_t);
    static size_t configured = 0;
    if (smem > 48 * 1024 && configured < smem) {
        cudaFuncSetAttribute(rerank_diff_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    cudaError_t e = launch_pdl(rerank_diff_kernel, dim3((heads + kRecycleWarps - 1) / kRecycleWarps),
                               dim3(kRecycleWarps * 32), smem, st, s, layer, old_sel, n_old, unstable, period,
                               force_due, old_has_tail, extra_tokens, slow_resident, row_skip, copies, max_copies,
                               n_copies, ws, batch);
    if (e != cudaSuccess) return e;
    return launch_pdl(rerank_commit_kernel, dim3(1), dim3(1024), 0, st, s, layer, copies, max_copies, n_copies, ws,
                      batch);
}

cudaError_t launch_fetch(const StoreView &s, int layer, const void *host_pages, const int32_t *copies,
                         const int32_t *n_copies, int max_copies, int page_bytes, const int32_t *staged_map,
                         const void *staging, int32_t *n_staged_hits, cudaStream_t st, int max_ctas, int row) {
    // inside a step (the rerank waits for it): one CTA per page, up to 8 per SM;
    // in the background: max_ctas
    const int grid = max(1, min(max_copies, max_ctas > 0 ? max_ctas : 148 * 8));
    return launch_pdl(fetch_kernel, dim3(grid), dim3(kCopyThreads), 0, st, s, layer, (const char *)host_pages,
                      copies, n_copies, max_copies, page_bytes, staged_map, (const char *)staging, n_staged_hits,
                      row);
}

cudaError_t launch_stage_plan(const StoreView &s, const int32_t *pred_sel, const int32_t *pred_n,
                              const uint8_t *unstable, const uint8_t *slow_resident, int32_t *staged_map,
                              int32_t *stage_list, int32_t *stage_count, int cap, int batch, int pass,
                              cudaStream_t st) {
    if (pass < 0 || pass >= kStagePasses) return cudaErrorInvalidValue;
    const int warps = batch * s.L * s.H;
    stage_mark_kernel<<<1, 1, 0, st>>>(stage_count, 1 + 2 * pass);
    if (warps > 0)
        stage_plan_kernel<<<(warps + 7) / 8, 256, 0, st>>>(s, pred_sel, pred_n, unstable, slow_resident,
                                                          staged_map, stage_list, stage_count, cap, batch);
    stage_mark_kernel<<<1, 1, 0, st>>>(stage_count, 2 + 2 * pass);
    return cudaGetLastError();
}

// a few CTAs only: the copies run beside decode and must not take its SMs
// (each CTA keeps 8 KiB of host reads in flight; 24 CTAs saturate the link)
#ifndef FC_STAGE_CTAS
#define FC_STAGE_CTAS 24
#endif
cudaError_t launch_stage_fetch(const StoreView &s, const void *host_pages, const int32_t *stage_list,
                               const int32_t *stage_count, int cap, void *staging, int page_bytes, int pass,
                               cudaStream_t st) {
    if (pass < 0 || pass >= kStagePasses) return cudaErrorInvalidValue;
    stage_fetch_kernel<<<max(1, min(cap, FC_STAGE_CTAS)), kCopyThreads, 0, st>>>(
        s, (const char *)host_pages, stage_list, stage_count, cap, (char *)staging, page_bytes, pass);
    return cudaGetLastError();
}

cudaError_t launch_stage(const StoreView &s, const int32_t *pred_sel, const int32_t *pred_n,
                         const uint8_t *unstable, const uint8_t *slow_resident, int32_t *staged_map,
                         int32_t *stage_list, int32_t *stage_count, int cap, const void *host_pages, void *staging,
                         int page_bytes, int batch, cudaStream_t st) {
    cudaError_t e = launch_stage_plan(s, pred_sel, pred_n, unstable, slow_resident, staged_map, stage_list,
                                      stage_count, cap, batch, 0, st);
    if (e != cudaSuccess) return e;
    return launch_stage_fetch(s, host_pages, stage_list, stage_count, cap, staging, page_bytes, 0, st);
}

cudaError_t launch_stage_clear(const StoreView &s, int32_t *staged_map, const int32_t *stage_list,
                               int32_t *stage_count, int cap, cudaStream_t st) {
    stage_clear_kernel<<<1, 1024, 0, st>>>(s, staged_map, stage_list, stage_count, cap);
    return cudaGetLastError();
}

cudaError_t launch_offload_filled(const StoreView &s, void *host_pages, const uint8_t *unstable,
                                  uint8_t *slow_resident, int batch, int page_bytes, cudaStream_t st) {
    const int grid = max(1, min(batch * s.L * s.H, 148 * 8));
    offload_filled_kernel<<<grid, kCopyThreads, 0, st>>>(s, (char *)host_pages, unstable, slow_resident,
                                                          batch, page_bytes);
    return cudaGetLastError();
}

cudaError_t launch_evict_unselected(const StoreView &s, const uint8_t *unstable, int batch, int extra,
                                    cudaStream_t st) {
    if (batch * s.L * s.H == 0) return cudaSuccess;
    evict_unselected_kernel<<<batch * s.L * s.H, 256, 0, st>>>(s, unstable, batch, extra);
    return cudaGetLastError();
}

cudaError_t launch_offload(const StoreView &s, void *host_pages, const int32_t *pages, int n,
                           int page_bytes, int max_ctas, cudaStream_t st) {
    const int grid = max(1, min(n, max_ctas > 0 ? max_ctas : 148 * 8));
    offload_kernel<<<grid, kCopyThreads, 0, st>>>(s, (char *)host_pages, pages, n, page_bytes);
    return cudaGetLastError();
}

}  // namespace fc
