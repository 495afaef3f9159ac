"""DecodeEngine: the per-decode-step KV hot path for a batch of requests.

This is the batched, GPU-resident counterpart of what the reference composes
per head in Python (attention.sparsity_error, attention.py:150-159) and
schedules in its simulator (simulator._decode_step / _append_token / _rerank,
simulator.py:410-547).  One decode step over L layers is, per layer:

  1. fc_score_select   for due heads only (unstable every step, stable at
                       t % R == 0; layers with no due head are skipped —
                       layer_scoring_skippable, scoring.py:205-209): group
                       page scores + exact top-K with the last page pinned
                       (subsystem 2)
  2. fc_sparse_decode  GQA split-K attention over sel ∪ pages appended since
                       the head's last rerank, combine fused (subsystem 3),
                       with the append fused in: the CTA staging a head's
                       last page writes the new token's k/v into it and folds
                       the key into the page's min/max summary (subsystem 1)

then fc_step_advance (seq_len += 1; new pages allocated from the device free
list).  Steps are replayed from CUDA graphs (one for rerank steps, one for
plain steps) so the <= 2·L+1 launches cost no host time.
"""

from __future__ import annotations

import gc
import math

import torch

from .config import HeadId
from .scoring import layer_scoring_skippable
from .stability import HeadProfile
from ._lib import FC_HOLD_NONE as HOLD_NONE, FC_HOLD_RERANK as HOLD_RERANK
from ._lib import FC_HOLD_RESUME as HOLD_RESUME, FC_HOLD_WAIT as HOLD_WAIT
from .store import PAGE_SIZE, KVStore
from . import _lib


class DecodeEngine:
    def __init__(self, *, batch: int, layers: int, kv_heads: int, group: int, head_dim: int,
                 ctx_cap_tokens: int, topk_pages: int, rerank_period: int,
                 profile: HeadProfile, dtype=torch.bfloat16, device="cuda",
                 n_blocks: int | None = None, tiering: bool = False, after_layer=None):
        if profile.n_layers != layers or profile.n_heads_per_layer != kv_heads:
            raise ValueError("profile grid does not match (layers, kv_heads)")
        self.B, self.L, self.H, self.G, self.D = batch, layers, kv_heads, group, head_dim
        self.K, self.R = topk_pages, rerank_period
        self.profile = profile
        self.device = torch.device(device)
        pages_cap = ctx_cap_tokens // PAGE_SIZE + 1
        if n_blocks is None:  # full residency: every page of every head has a block
            n_blocks = batch * layers * kv_heads * pages_cap + 1
        self.sel_slack = rerank_period // PAGE_SIZE + 2  # pages appended between reranks
        self.store = KVStore(batch_cap=batch, layers=layers, kv_heads=kv_heads, group=group,
                             head_dim=head_dim, pages_cap=pages_cap, n_blocks=n_blocks,
                             sel_cap=topk_pages + self.sel_slack, dtype=dtype, device=self.device)
        self.unstable = profile.mask_tensor(self.device).contiguous()
        self.t = 1                # host mirror of store.step: the upcoming decode step
        self.selected = False     # initial selection done (made at the first step)
        self.seq_host = [0] * batch
        # per-request decode state (host mirrors of store.row_phase / row_hold):
        # row b's own step is t_b = t + phase[b] (simulator.py:437-439); rows
        # admitted together share a phase, rows admitted later rerank on their
        # own boundary
        self.phase = [0] * batch
        self.hold = [0] * batch
        self._hold_host = torch.zeros(batch, dtype=torch.uint8, pin_memory=True)
        self._hold_dev_state = [0] * batch  # what the device buffer holds
        self.decoded_rows: list[int] = []   # rows that emitted a token at the last step
        self.rerank_rows: list[int] = []    # rows at their rerank boundary at the last step
        self._initial_rows: set = set()     # admitted rows whose initial selection is due
        self.att_bound = min(pages_cap, topk_pages + self.sel_slack)
        # static step buffers (CUDA-graph inputs/outputs)
        Hq = kv_heads * group
        self.q = torch.zeros((layers, batch, Hq, head_dim), dtype=dtype, device=self.device)
        self.k_new = torch.zeros((layers, batch, kv_heads, head_dim), dtype=dtype, device=self.device)
        self.v_new = torch.zeros_like(self.k_new)
        self.out = torch.zeros_like(self.q)
        self._graphs: dict[tuple, torch.cuda.CUDAGraph] = {}  # (kind, score_all_heads)
        # per-layer hook after the attention launch (e.g. the head-sharded
        # all-gather of outputs, dist.HeadGroup); captured into the step graph
        self.after_layer = after_layer
        # attention of heads a layer's scoring launch does not select starts
        # without waiting for it (fc_sparse_decode early_unstable)
        self.early_heads = True
        # attention as persistent launches over runs of layers with no scoring /
        # recycle between them (fc_sparse_decode_layers) — True / False, or
        # None = auto: where the per-head persistent kernel splits heads over
        # clusters (<= 74 heads per layer on 148 SMs; measured 1.6x faster
        # steps at batch 1, 9 % at batch 4), per-layer launches above (equal
        # or 2 % faster at config 2)
        self.run_kernel = None
        # scored layers run scoring, selection and attention in one launch (one
        # CTA per head, fc_score_attend) when the batch fills the GPU with
        # heads: 53.4 vs 56.6 us per scored layer at config 2
        self.fused_score_attend = True
        # plain steps of fused layers: the heads scored every step (unstable)
        # get a cluster of CTAs each and the others one CTA each, when the
        # bandwidth model says the uniform split is unbalanced (small batches
        # at long context: config 4; fc_score_attend_map)
        self.mixed_clusters = True
        self._mixed: dict = {}
        # 'partial' steps (some rows at their boundary): the heads due in a
        # layer get a cluster of CTAs each, the others one CTA each, with the
        # map rewritten before each step for the rows due then (a static
        # device buffer per layer pattern, so one graph serves every step)
        self.partial_clusters = True
        self._partial: dict = {}      # unstable-head pattern -> (S, n_ctas, buffer) or None
        self._partial_maps: dict = {}  # (pattern, due rows) -> device map
        # plain steps of layers where only some heads are due (the unstable
        # heads spread over the layers): the due heads' scoring spread over
        # every SM, then one CTA per head selects and attends
        # (fc_score_attend_balanced; 37.5 vs 45 us per layer at config 2 with
        # 2 of 8 KV heads unstable)
        self.balanced_scoring = True
        # profiling: score every head every step and record
        # the selections on the device (trace.TraceRecorder)
        self.score_all_heads = False
        self.recorder = None
        # two-tier mode (subsystem 4): stable heads keep only their selection in
        # HBM; every full page lives once in the pinned host tier
        self.tiering = tiering
        self.tier = None
        self.stager = None
        if tiering:
            from .tiering import TierStore
            self.tier = TierStore(self.store, profile)
            st = self.store
            # per layer (layer-major so each layer's slice is contiguous): the
            # resident set before the rerank, the copy list and its length
            self.old_sel = torch.zeros((layers, batch, kv_heads, st.SELCAP), dtype=torch.int32,
                                       device=self.device)
            self.n_old = torch.zeros((layers, batch, kv_heads), dtype=torch.int32, device=self.device)
            self.copies = torch.zeros((layers, batch * kv_heads * st.SELCAP, 4), dtype=torch.int32,
                                      device=self.device)
            self.n_copies = torch.zeros(layers, dtype=torch.int32, device=self.device)
            self.fetched_pages = torch.zeros(1, dtype=torch.int64, device=self.device)
            # reload pauses: one recycle of every layer after the step's attention
            # (the rows it touches are held) and one copy list for the fetch stream
            self.old_sel_all = torch.zeros_like(st.sel)
            self.n_old_all = torch.zeros_like(st.n_sel)
            self.copies_all = torch.zeros((batch * layers * kv_heads * st.SELCAP, 4), dtype=torch.int32,
                                          device=self.device)
            self.n_copies_all = torch.zeros(1, dtype=torch.int32, device=self.device)
            self._stable_layers = [l for l in range(layers)
                                   if any(not profile.is_unstable(HeadId(l, h)) for h in range(kv_heads))]
            # promoted pages staged on a side stream `lead` steps before each
            # rerank (tiering.ReloadStager); None: every promotion crosses the
            # host link inside the rerank step
            from .tiering import ReloadStager
            self.stager = ReloadStager(self.store, self.tier, self.unstable, topk_pages,
                                       leads=(min(2, max(1, rerank_period - 1)),))
            # serving (admit): the post-prefill offload runs on a side stream; a
            # row keeps every page, and reranks skip it (row_skip), until that
            # copy has finished — then its unselected stable-head pages are
            # evicted (simulator.py:389-408 releases them at offload end)
            self.row_skip = torch.zeros(batch, dtype=torch.uint8, device=self.device)
            self.offload_stream = None
            self._evict_pending: dict[int, tuple] = {}  # row -> (offload done event, step admitted)
            self.evict_hold_steps = 0  # test hook: keep an eviction pending at least this many steps
            # CTAs of that background copy: the rest of the GPU keeps decoding
            self.offload_ctas = 16
            # reload pause (simulator.py:321-323,542): a row's
            # promoted pages are fetched on a side stream after its rerank step;
            # the row is held (no attention, no advance) until they landed while
            # the other rows keep decoding.  Off: the fetch runs inside the step.
            self.reload_pause = False
            self.fetch_stream = None
            self.fetch_ctas = 32  # (51 GB/s from 32 CTAs, scripts/micro/fetch_bw.cu)
            self.fetch_log = None  # list: (start, end, pages) of each background fetch (profiling)
            self._reloads: dict[int, torch.cuda.Event] = {}  # row -> fetch done
            self._snap_free: list[torch.Tensor] = []
            self._snap_busy: list[tuple] = []                # (event, copies snapshot)

    # -- prefill ----------------------------------------------------------------

    def prefill(self, row: int, keys: torch.Tensor, values: torch.Tensor) -> None:
        """keys/values [L, H, T, d] (any device): allocate pages for positions
        0..T (the next decode position included) and write them with their
        summaries (build_minmax, scoring.py:72-90)."""
        L, H, T, d = keys.shape
        self.store.alloc_pages(row, 0, T // PAGE_SIZE + 1)
        for layer in range(L):
            self.store.prefill(row, layer, keys[layer], values[layer])
        self.store.seq_len[row] = T
        self.seq_host[row] = T

    # -- rows joining and leaving (serving loop, f4) -------------------------------

    def start_serving(self) -> None:
        """Every row free (seq_len = -1: skipped by every kernel); requests
        then join with admit() and leave with retire()."""
        self.store.seq_len.fill_(-1)
        self.seq_host = [-1] * self.B
        self.selected = True            # initial selections are made per admitted row
        # requests join at any step: their phases differ, so the kernels always
        # read the per-request state (the step graphs captured at the first
        # admission then serve every later step)
        self._serving = True
        self._initial_rows = set()
        if self.stager is not None:
            # a batch of rows reranks together: each rerank moves many pages
            # over the host link, so predict R/2 steps ahead to give the
            # staging copy time (16 rows, R = 16: p95 TPOT 19 -> 10 ms,
            # 2.4k -> 2.7-3.2k tokens/s with rho = 0.99 queries)
            self.stager.leads = (max(1, self.R // 2),)
            self.stager.lead = self.stager.leads[0]

    def admit(self, row: int, keys: torch.Tensor, values: torch.Tensor) -> None:
        """Prefill request row ``row`` (keys/values [L, H, T, d]); its initial
        selection is made at its first decode step, with that step's query."""
        if self.seq_host[row] >= 0:
            raise ValueError(f"row {row} is busy")
        self.prefill(row, keys, values)
        # the request's own step counter starts here: its first decode step is
        # t = 1 (simulator.py:437-439), whatever the engine's global step
        self.set_row_step(row, 1)
        self._set_hold(row, HOLD_NONE)
        if self.tiering:
            # post-prefill offload of every full stable-head page, in the
            # background (tiering.py:122-139): decode steps continue meanwhile
            cur = torch.cuda.current_stream(self.device)
            if self.offload_stream is None:
                self.offload_stream = torch.cuda.Stream(self.device)
            self.offload_stream.wait_stream(cur)
            with torch.cuda.stream(self.offload_stream):
                self.tier.offload_after_prefill(row, keys.shape[2] // PAGE_SIZE, self.offload_ctas)
                done = torch.cuda.Event()
                done.record()
            self.row_skip[row] = 1
            self._evict_pending[row] = (done, self.t)
        self._initial_rows.add(row)

    def eviction_pending(self, row: int) -> bool:
        """True while ``row`` still holds every page (its post-prefill
        offload has not finished, or its initial selection is not made)."""
        return self.tiering and row in self._evict_pending

    def _drain_evictions(self) -> None:
        # rows whose offload finished and whose initial selection exists keep
        # only their selection from now on (in stream order before this step)
        cur = torch.cuda.current_stream(self.device)
        for row, (done, t0) in list(self._evict_pending.items()):
            if row in self._initial_rows or self.t - t0 < self.evict_hold_steps or not done.query():
                continue
            cur.wait_event(done)
            self.store.evict_unselected_row(row, self.unstable)
            self.row_skip[row] = 0
            del self._evict_pending[row]

    def retire(self, row: int) -> None:
        """A finished request: every page of its row back to the free list."""
        if self.tiering and row in self._evict_pending:  # its blocks may still be read by the offload
            torch.cuda.current_stream(self.device).wait_event(self._evict_pending.pop(row)[0])
            self.row_skip[row] = 0
        if self.tiering and row in self._reloads:  # its blocks may still be written by the fetch
            torch.cuda.current_stream(self.device).wait_event(self._reloads.pop(row))
        self._set_hold(row, HOLD_NONE)
        if self.stager is not None:
            self.stager.forget_row(row)
        self.store.free_row(row)
        self.seq_host[row] = -1
        self._initial_rows.discard(row)
        if self.tiering:
            self.tier.release_row(row)

    def _initial_selections(self) -> None:
        # every head of a newly admitted row selects with this step's query
        # (the batch graph then re-scores only the heads that are due)
        for row in sorted(self._initial_rows):
            for layer in range(self.L):
                self.store.score_select_row(row, layer, self.q[layer, row], self.unstable, self.R, self.K,
                                            force_due=True, extra_tokens=1)
        self._initial_rows.clear()
        # (two-tier: stable heads keep only their selection once the
        # post-prefill offload is done, _drain_evictions)

    def prefill_layer(self, row: int, layer: int, k: torch.Tensor, v: torch.Tensor,
                      alloc: bool) -> None:
        """Layer-at-a-time prefill (bench scale); ``alloc`` on the first layer."""
        T = k.shape[1]
        if alloc:
            self.store.alloc_pages(row, 0, T // PAGE_SIZE + 1)
        self.store.prefill(row, layer, k, v)
        self.store.seq_len[row] = T
        self.seq_host[row] = T

    # -- per-request steps and reload pauses -------------------------------------------

    def row_t(self, row: int, t: int | None = None) -> int:
        """Row ``row``'s own decode step at global step ``t`` (default: the upcoming one)."""
        return (self.t if t is None else t) + self.phase[row]

    def set_row_step(self, row: int, t_row: int) -> None:
        """Make row ``row``'s upcoming decode step ``t_row``: it reranks when its
        own step is a multiple of R (its rerank phase)."""
        self.phase[row] = int(t_row) - self.t
        self.store.row_phase[row] = self.phase[row]

    def _set_hold(self, row: int, mode: int) -> None:
        self.hold[row] = mode

    def _sync_holds(self) -> None:
        # the device copy of the hold modes, for the step about to launch (a
        # small H2D from a ring of pinned buffers, in stream order)
        if self.hold == self._hold_dev_state:
            return
        ring = self.__dict__.setdefault("_hold_ring", [])
        if len(ring) < 4:
            buf = (torch.zeros(self.B, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
            ring.append(buf)
        else:
            buf = ring.pop(0)
            ring.append(buf)
            buf[1].synchronize()  # its last copy has been consumed
        buf[0].copy_(torch.tensor(self.hold, dtype=torch.uint8))
        self.store.row_hold.copy_(buf[0], non_blocking=True)
        buf[1].record()
        self._hold_dev_state = list(self.hold)

    def _active_rows(self):
        return [b for b in range(self.B) if self.seq_host[b] >= 0]

    def boundary_rows(self, t: int | None = None) -> list:
        """Rows whose stable heads are due at global step ``t`` (their own step
        is a multiple of R); at the upcoming step, rows waiting for or resuming
        after a reload are not (their selection for t_b exists)."""
        now = t is None or t == self.t
        t = self.t if t is None else t
        return [b for b in self._active_rows()
                if (t + self.phase[b]) % self.R == 0 and not (now and self.hold[b] in (HOLD_WAIT, HOLD_RESUME))]

    def step_kind(self, t: int | None = None) -> str:
        """'plain' (no row at its boundary), 'rerank' (every decoding row) or
        'partial' (some rows: requests at different phases)."""
        now = t is None or t == self.t
        due = self.boundary_rows(t)
        if not due:
            return "plain"
        rows = [b for b in self._active_rows() if not (now and self.hold[b] == HOLD_WAIT)]
        return "rerank" if len(due) == len(rows) else "partial"

    def is_rerank_step(self, t: int | None = None) -> bool:
        """Some row reranks at global step ``t`` (default: the upcoming one)."""
        return self.step_kind(t) != "plain"

    def _per_row_needed(self) -> bool:
        # the kernels read the per-request state only when some active row is
        # out of phase with the global step or rows can be held
        return (getattr(self, "_serving", False) or (self.tiering and self.reload_pause)
                or any(self.phase[b] != 0 for b in self._active_rows()))

    def _phases_aligned(self) -> bool:
        ph = {self.phase[b] % self.R for b in self._active_rows()}
        return len(ph) <= 1

    def _fetch_mode(self) -> str:
        """How a two-tier rerank fetches promoted pages: 'async' (side stream,
        the row held), 'staged' (predicted pages staged ahead, the rest inside
        the step; rows in phase only) or 'inline' (inside the step)."""
        if not self.tiering:
            return "inline"
        if self.reload_pause:
            return "async"
        if self.stager is not None and self._phases_aligned():
            return "staged"
        return "inline"

    def _plan_holds(self) -> None:
        if not (self.tiering and self.reload_pause):
            for b in range(self.B):
                self.hold[b] = HOLD_NONE
            return
        for b in range(self.B):
            if self.seq_host[b] < 0:
                self.hold[b] = HOLD_NONE
            elif b in self._reloads:
                if self._reloads[b].query():
                    del self._reloads[b]
                    self.hold[b] = HOLD_RESUME
                else:
                    self.hold[b] = HOLD_WAIT
            elif (self.row_t(b) % self.R == 0 and self._stable_layers and not self.eviction_pending(b)):
                self.hold[b] = HOLD_RERANK
            else:
                self.hold[b] = HOLD_NONE

    def _launch_reloads(self) -> None:
        """After a step graph with reranking rows held: fetch their promoted
        pages on the fetch stream (from a snapshot of the copy lists, which the
        next step's recycles overwrite); the rows resume once it finished."""
        rows = [b for b in range(self.B) if self.hold[b] == HOLD_RERANK]
        if not rows:
            return
        dev = self.device
        main = torch.cuda.current_stream(dev)
        if self.fetch_stream is None:
            # the fetch kernel is a handful of CTAs that mostly wait on the host
            # link; at high priority they take the next free SMs rather than
            # queueing behind the back-to-back decode launches
            self.fetch_stream = torch.cuda.Stream(dev, priority=-5)
        busy = []
        for ev, snap in self._snap_busy:
            if ev.query():
                self._snap_free.append(snap)
            else:
                busy.append((ev, snap))
        self._snap_busy = busy
        snap = self._snap_free.pop() if self._snap_free else (torch.empty_like(self.copies_all),
                                                              torch.empty_like(self.n_copies_all))
        snap[0].copy_(self.copies_all)
        snap[1].copy_(self.n_copies_all)
        ready = torch.cuda.Event()
        ready.record(main)
        with torch.cuda.stream(self.fetch_stream):
            self.fetch_stream.wait_event(ready)
            # one launch per row, in row order: each row resumes as soon as its
            # own pages landed (a single launch for all made rows that reranked
            # together resume together and rerank together again: the phases
            # clumped and the host link idled between clumps)
            t0 = None
            if self.fetch_log is not None:
                t0 = torch.cuda.Event(enable_timing=True)
                t0.record(self.fetch_stream)
            for b in rows:
                self.store.fetch_pages_all_layers(self.tier.host, snap[0], snap[1], self.fetch_ctas, row=b)
                done = torch.cuda.Event(enable_timing=t0 is not None)
                done.record(self.fetch_stream)
                self._reloads[b] = done
            if t0 is not None:  # (instrumentation: fetch duration and pages per step)
                n = torch.empty(1, dtype=torch.int32, device=self.device)
                n.copy_(snap[1])
                self.fetch_log.append((t0, done, n))
        self._snap_busy.append((done, snap))

    # -- one decode step -----------------------------------------------------------

    def _launch_step(self, kind: str, force_due: bool, fetch: str = "inline") -> None:
        st = self.store
        tiered_rerank = self.tiering and kind != "plain" and not force_due
        # reload pauses: the rows that rerank are held this step, so their
        # recycle (every layer, one launch) runs after the other rows' attention
        # and their fetch on the fetch stream (_launch_reloads); the layers
        # launch as at a step without recycles
        deferred = tiered_rerank and fetch == "async"
        use_run = self._use_run()
        use_fused = self.fused_score_attend and st.score_attend_supported(self.B)

        def recycles(l):
            return tiered_rerank and not deferred and l in self._stable_layers

        def scores(l):
            return force_due or not self._layer_skippable(l, kind)

        if deferred:  # resident set of stable heads = their current selection
            self.old_sel_all.copy_(st.sel)
            self.n_old_all.copy_(st.n_sel)
            self.n_copies_all.zero_()
        elif tiered_rerank:
            self.old_sel.copy_(st.sel.transpose(0, 1))
            self.n_old.copy_(st.n_sel.transpose(0, 1))
            self.n_copies.zero_()
        layer = 0
        _lib.capture_probe(f"{kind} step prologue")
        while layer < self.L:
            _lib.capture_probe(f"{kind} step, before layer {layer}")
            recycle = recycles(layer)
            scored = scores(layer)
            if scored and not recycle and self._use_balanced(layer, kind, force_due):
                st.score_attend_balanced(layer, self.q[layer], self.unstable, self.R, self.K, self.out[layer],
                                         self.B, extra_tokens=1, kv_prefetch=layer > 0, k_new=self.k_new[layer],
                                         v_new=self.v_new[layer], attend_appended=False)
                if self.after_layer is not None:
                    self.after_layer(layer)
                layer += 1
                continue
            if scored and not recycle and use_fused:
                # one launch: every head's CTA scores, selects and attends
                plan = None
                if kind == "plain" and not force_due:
                    plan = self._mixed_plan(layer)
                elif kind == "partial" and not force_due:
                    # (where the balanced launch is not used: 35.4 vs 33.9 us per
                    # layer at config 2 with one row of 16 due, partial_probe.py)
                    plan = self._partial_plan(layer)
                st.score_attend(layer, self.q[layer], self.unstable, self.R, self.K, self.out[layer], self.B,
                                force_due=force_due, extra_tokens=1, kv_prefetch=layer > 0,
                                k_new=self.k_new[layer], v_new=self.v_new[layer], attend_appended=False,
                                cta_map=plan[0] if plan else None, cluster=plan[1] if plan else 0)
                if self.after_layer is not None:
                    self.after_layer(layer)
                layer += 1
                continue
            if scored:
                # the previous kernel (the last layer's attention) never writes this
                # layer's summaries / selection: plan and warm L2 while it drains
                st.score_select(layer, self.q[layer], self.unstable, self.R, self.K, self.B,
                                force_due=force_due, extra_tokens=1, kv_prefetch=layer > 0)
            if recycle:  # fused diff/recycle, then fetch the promoted pages over PCIe
                nc = self.n_copies[layer:layer + 1]
                st.rerank_recycle(layer, self.old_sel[layer], self.n_old[layer], self.unstable, self.R,
                                  self.copies[layer], nc, self.B, old_has_tail=False, extra_tokens=1,
                                  slow_resident=self.tier.slow_resident, row_skip=self.row_skip)
                if fetch == "staged":
                    self.stager.fetch(layer, self.copies[layer], nc)
                elif fetch == "inline":
                    self.tier.reload(layer, self.copies[layer], nc)
                # ("async": the rows are held; _launch_reloads fetches after the step)
            if use_run:
                # persistent attention over the run of layers up to the next one
                # that needs a selection / table update (or a per-layer hook)
                end = layer + 1
                if self.after_layer is None:
                    while end < self.L and not (scores(end) or recycles(end)):
                        end += 1
                st.sparse_decode_layers(layer, end - layer, self.q[layer:end], self.out[layer:end], self.B,
                                        max_pages=self.att_bound, extra_tokens=1, attend_appended=False,
                                        k_new=self.k_new[layer:end], v_new=self.v_new[layer:end],
                                        first_dep=scored or recycle or layer == 0)
                if self.after_layer is not None:
                    self.after_layer(layer)
                layer = end
                continue
            # with no scoring / recycle launch in this layer, the previous kernel
            # (the last layer's attention, or the step advance) does not touch
            # this layer's selection, table or pages: stage KV while it drains
            st.sparse_decode(layer, self.q[layer], self.out[layer], self.B,
                             max_pages=self.att_bound, extra_tokens=1, attend_appended=False,
                             k_new=self.k_new[layer], v_new=self.v_new[layer],
                             kv_prefetch=not (scored or recycle) and self.after_layer is None and layer > 0,
                             # heads the scoring launch leaves alone overlap it
                             early_unstable=self.unstable if scored and not recycle and not force_due
                             and self.early_heads else None, early_period=self.R)
            if self.after_layer is not None:
                self.after_layer(layer)
            layer += 1
        if deferred:
            st.rerank_recycle_all_layers(self.old_sel_all, self.n_old_all, self.unstable, self.R, self.copies_all,
                                         self.n_copies_all, self.B, slow_resident=self.tier.slow_resident,
                                         row_skip=self.row_skip)
            self.fetched_pages.add_(self.n_copies_all.sum())
        elif tiered_rerank:
            self.fetched_pages.add_(self.n_copies.sum())
            if fetch == "staged":
                self.stager.finish_rerank()
        st.step_advance(self.B, self.unstable, self.R)
        if self.recorder is not None:
            self.recorder.capture()
        if self.tiering:  # write-once offload of the page that just filled
            st.offload_filled(self.tier.host, self.unstable, self.tier.slow_resident, self.B)

    def _use_balanced(self, layer: int, kind: str, force_due: bool) -> bool:
        # some but not all of the layer's heads due: a plain step of a layer
        # with a few unstable heads, or a step where some rows are at their
        # rerank boundary (requests at different phases)
        if not self.balanced_scoring or kind == "rerank" or force_due:
            return False
        n_unst = sum(self.profile.is_unstable(HeadId(layer, h)) for h in range(self.H))
        if kind == "plain" and n_unst == 0:
            return False
        if n_unst == self.H:  # every head due at every step: the fused launch
            return False
        # (only where the fused kernel gives every head one CTA: smaller batches
        # split heads over clusters, and config 4's mixed clusters beat this
        # there: 6.1k vs 5.1k tokens/s)
        return (self.store.score_attend_supported(self.B) == 1
                and self.store.score_attend_balanced_supported(self.B) > 0)

    def _mixed_plan(self, layer: int):
        # heads due at a plain step = the layer's unstable heads; the map is
        # sized for the current longest row (any map gives the same results)
        if not self.mixed_clusters:
            return None
        if layer not in self._mixed:
            scored = [h for h in range(self.H) if self.profile.is_unstable(HeadId(layer, h))]
            n_pages = (max(self.seq_host) + 1 + PAGE_SIZE - 1) // PAGE_SIZE
            self._mixed[layer] = (self.store.mixed_cluster_map(self.B, scored, n_pages, self.K)
                                  if scored and n_pages > 0 else None)
        return self._mixed[layer]

    def _layer_pattern(self, layer: int) -> tuple:
        return tuple(h for h in range(self.H) if self.profile.is_unstable(HeadId(layer, h)))

    def _partial_plan(self, layer: int):
        """(map buffer, S) for a 'partial' step's fused launch of ``layer``,
        or None (balanced / uniform launch instead).  Sized for the most rows
        at their boundary on one step under the current phases."""
        if not (self.partial_clusters and self.fused_score_attend and self.store.score_attend_supported(self.B)):
            return None
        pat = self._layer_pattern(layer)
        if len(pat) == self.H:
            return None
        if pat not in self._partial:
            rows = self._active_rows()
            per_res = {}
            for b in rows:
                per_res[(self.t + self.phase[b]) % self.R] = per_res.get((self.t + self.phase[b]) % self.R, 0) + 1
            max_due = max(per_res.values()) if per_res else 1
            n_s = len(rows) * len(pat) + max_due * (self.H - len(pat))
            n_pages = (max(self.seq_host) + 1 + PAGE_SIZE - 1) // PAGE_SIZE
            # (per-CTA rate and selection latency as measured for a scored head
            # at config 2: ~45 GB/s, ~7 us from streamed to attending,
            # scripts/partial_probe.py)
            plan = (self.store.cluster_plan(self.B, n_s, n_pages, self.K, bw_sm_gbs=45.0, select_us=7.0)
                    if n_pages > 0 else None)
            if plan is not None:
                S, n_ctas = plan
                plan = (S, n_ctas, torch.full((n_ctas,), -1, dtype=torch.int32, device=self.device))
            self._partial[pat] = plan
        p = self._partial[pat]
        return None if p is None else (p[2], p[0])

    def _fill_partial_maps(self) -> None:
        # the CTA maps of this step's due (row, head) pairs into the static buffers
        due = tuple(self.boundary_rows())
        active = self._active_rows()
        for pat, plan in self._partial.items():
            if plan is None:
                continue
            key = (pat, due)
            m = self._partial_maps.get(key)
            if m is None:
                scored = {(b, h) for b in active for h in pat if self.hold[b] != HOLD_WAIT}
                scored |= {(b, h) for b in due for h in range(self.H)}
                S, n_ctas, _ = plan
                if len(self._partial_maps) > 4096:
                    self._partial_maps.clear()
                m = self._partial_maps[key] = self.store.cluster_map_pairs(self.B, scored, S, n_ctas).to(
                    self.device)
            plan[2].copy_(m, non_blocking=True)

    def _use_run(self) -> bool:
        if self.run_kernel is None:
            return self.store.run_split(self.B, self.att_bound) >= 2
        return bool(self.run_kernel) and self.store.run_supported(self.B, self.att_bound)

    def _layer_skippable(self, layer: int, kind: str) -> bool:
        # a representative step of the same kind: R (some row reranks) or 1
        # (plain, R > 1)
        t = self.R if kind != "plain" else (1 if self.R > 1 else self.R)
        return layer_scoring_skippable(layer, t, self.profile, self.R)

    def _initial_selection(self) -> None:
        # every head selects with the first step's query (the selection a
        # request enters decode with; not a scheduled score evaluation, so the
        # step's own scoring of its due heads follows as at any step)
        if self.tiering:  # post-prefill offload of every full stable-head page
            for b in range(self.B):
                self.tier.offload_after_prefill(b, self.seq_host[b] // PAGE_SIZE)
        for layer in range(self.L):
            self.store.score_select(layer, self.q[layer], self.unstable, self.R, self.K, self.B,
                                    force_due=True, extra_tokens=1, counted=False)
        if self.tiering:  # keep only the selection of stable heads in HBM
            self.store.evict_unselected(self.unstable, self.B)

    def step(self, *, use_graph: bool = True) -> torch.Tensor:
        """Run one decode step on the engine's static buffers (q, k_new,
        v_new -> out).  The first step after prefill first makes the initial
        selection of every head.  Rows at their own rerank boundary rerank;
        with ``reload_pause`` a two-tier row is held from its rerank until its
        promoted pages landed (``decoded_rows``: the rows that emitted)."""
        if not self.selected:
            self._initial_selection()
            self.selected = True
            use_graph = False  # (eager: sizes the workspaces the graphs capture)
        if self._initial_rows:
            self._initial_selections()
        if self.tiering and self._evict_pending:
            self._drain_evictions()
        self.store.per_row = self._per_row_needed()
        self._plan_holds()
        self._sync_holds()
        kind = self.step_kind()
        fetch = self._fetch_mode()
        self.rerank_rows = self.boundary_rows()
        staged = kind != "plain" and fetch == "staged"
        if staged:
            self.stager.wait()  # staged promotions have landed
        if kind == "partial" and not self.score_all_heads:
            if not use_graph or (kind, False, fetch, self.store.per_row) not in self._graphs:
                for layer in range(self.L):  # plans (and their buffers) exist before launch / capture
                    self._partial_plan(layer)
            self._fill_partial_maps()
        if use_graph:
            key = (kind, self.score_all_heads, fetch, self.store.per_row)
            g = self._graphs.get(key)
            if g is None:
                g = self._capture(kind, fetch)
            g.replay()
        else:
            self._launch_step(kind, force_due=self.score_all_heads, fetch=fetch)
        if staged:
            self.stager.rerank_launched()
        if fetch == "async" and kind != "plain":
            self._launch_reloads()
        if fetch == "staged" and not self.score_all_heads:
            rows = self._active_rows()
            t0 = self.row_t(rows[0]) if rows else self.t
            if any((t0 + ld) % self.R == 0 for ld in self.stager.leads):
                self.stager.predict(self.q, self.B, self._stable_layers)
        self.decoded_rows = [b for b in self._active_rows() if self.hold[b] not in (HOLD_WAIT, HOLD_RERANK)]
        for b in self._active_rows():
            if self.hold[b] in (HOLD_WAIT, HOLD_RERANK):
                self.phase[b] -= 1  # (the device did the same in the step advance)
            else:
                self.seq_host[b] += 1
        self.t += 1
        return self.out

    def attach_recorder(self, recorder) -> None:
        """Record top-K traces from the next step on (every head scored every
        step while attached); ``None`` detaches.  Step graphs are re-captured."""
        self.recorder = recorder
        self.score_all_heads = recorder is not None
        self._graphs.clear()

    def capture_graphs(self, kinds=("plain", "rerank")) -> None:
        """Capture the step graphs of ``kinds`` now (with the current fetch
        mode), so no capture or instantiation happens inside a timed region."""
        fetch = self._fetch_mode()
        self.store.per_row = self._per_row_needed()
        for kind in kinds:
            if (kind, self.score_all_heads, fetch, self.store.per_row) not in self._graphs:
                self._capture(kind, fetch)

    def _capture(self, kind: str, fetch: str) -> torch.cuda.CUDAGraph:
        # stream capture records the launches without executing them, so the
        # engine state is untouched; workspaces were sized by the eager first step
        if kind == "plain":  # mixed-cluster maps live on the device: build them outside the capture
            for layer in range(self.L):
                self._mixed_plan(layer)
        if kind == "partial":
            for layer in range(self.L):
                self._partial_plan(layer)
        torch.cuda.synchronize(self.device)
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        # No garbage collection inside the capture: an unreachable engine of
        # an earlier request / test still holding its step graphs would have
        # them destroyed mid-capture (cudaGraphExecDestroy is not permitted
        # while a stream captures), which invalidates this capture.
        gc.collect()
        gc_was_enabled = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    self._launch_step(kind, force_due=self.score_all_heads, fetch=fetch)
        finally:
            if gc_was_enabled:
                gc.enable()
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        self._graphs[(kind, self.score_all_heads, fetch, self.store.per_row)] = g
        return g

    def launches_per_step(self, t: int) -> int:
        """Library kernel launches in the step graph for step t (mirrors
        _launch_step): per layer a scoring launch when a head is due and an
        attention launch (append fused) — one fused launch for both, or one
        persistent launch per run of layers, when those are enabled — plus
        the step advance (and the tier copies in two-tier mode)."""
        kind = self.step_kind(t)
        rerank = kind != "plain"
        st = self.store
        use_run = self._use_run()
        use_fused = self.fused_score_attend and st.score_attend_supported(self.B)
        fetch = self._fetch_mode()

        deferred = self.tiering and rerank and fetch == "async"

        def recycles(l):
            return self.tiering and rerank and not deferred and l in self._stable_layers

        def scores(l):
            return self.score_all_heads or not self._layer_skippable(l, kind)

        n, layer = 1, 0  # the step advance

        def recycle_kernels(heads):  # diff + commit, or one CTA for <= 32 heads (recycle.cu)
            return 1 if heads <= 32 and heads * 6 * (st.SELCAP + 64) * 4 <= 200 * 1024 else 2

        if deferred:
            # one recycle of every layer; one fetch per held row on the fetch stream
            n += recycle_kernels(self.B * self.L * self.H) + 1
        while layer < self.L:
            if recycles(layer):
                n += recycle_kernels(self.B * self.H) + 1  # recycle + fetch
            if scores(layer) and not recycles(layer) and (
                    use_fused or (not self.score_all_heads and self._use_balanced(layer, kind, False))):
                n += 1
                layer += 1
                continue
            n += 1 if scores(layer) else 0
            end = layer + 1
            if use_run and self.after_layer is None:
                while end < self.L and not (scores(end) or recycles(end)):
                    end += 1
            n += 1
            layer = end
        if self.tiering:
            n += 1  # offload of the page that just filled
            if rerank and fetch == "staged":
                n += 1  # staging map clear
        return n

    # -- host-buffer API (end-to-end path) -------------------------------------------

    def step_host(self, q_host: torch.Tensor, k_host: torch.Tensor, v_host: torch.Tensor,
                  out_host: torch.Tensor) -> None:
        """One step from pinned host inputs to a pinned host output: H2D of
        q/k/v, the step, D2H of the attention outputs, all on the current
        stream (asynchronous; the caller synchronises)."""
        self.q.copy_(q_host, non_blocking=True)
        self.k_new.copy_(k_host, non_blocking=True)
        self.v_new.copy_(v_host, non_blocking=True)
        self.step()
        out_host.copy_(self.out, non_blocking=True)

    def host_pipeline(self) -> "HostPipeline":
        return HostPipeline(self)

    # -- accounting ------------------------------------------------------------------

    def attended_pages(self) -> torch.Tensor:
        """[B, L, H] pages each head attends at the upcoming step (after its
        selection): n_sel + pages appended since the head's last rerank."""
        st = self.store
        n_tok = st.seq_len.long() + 1
        n_pages = (n_tok + PAGE_SIZE - 1) // PAGE_SIZE
        last = torch.gather(st.sel.long(), 3, (st.n_sel.long() - 1).clamp(min=0).unsqueeze(-1))[..., 0]
        last = torch.where(st.n_sel > 0, last, torch.full_like(last, -1))
        app = (n_pages[:, None, None] - 1 - last).clamp(min=0)
        return st.n_sel.long() + app

    def attention_bytes(self, layer: int) -> int:
        """Algorithmic HBM bytes of one fc_sparse_decode launch:
        K+V of the attended pages (the partial last page by its tokens) + the
        table and selection entries read + q and o."""
        st = self.store
        e = st.kv_pool.element_size()
        att = self.attended_pages()[:, layer]                      # [B, H]
        n_tok = st.seq_len.long() + 1
        last_fill = ((n_tok - 1) % PAGE_SIZE + 1)[:, None]          # tokens in the last page
        kv = ((att - 1) * PAGE_SIZE + last_fill) * 2 * self.D * e
        meta = att * 8                                              # table + sel entries
        qo = 2 * self.G * self.D * e
        return int((kv + meta + qo).sum().item())

    def scoring_bytes(self, layer: int, t: int) -> int:
        """Algorithmic bytes of fc_score_select at step t for one layer: the
        summaries of every scored page (all but the pinned last) + q."""
        st = self.store
        e = st.summaries.element_size()
        due = [self.profile.is_unstable(HeadId(layer, h)) or t % self.R == 0 for h in range(self.H)]
        n_pages = (st.seq_len.long() + 1 + PAGE_SIZE - 1) // PAGE_SIZE
        per_head = ((n_pages - 1) * 2 * self.D * e + self.G * self.D * e)
        return int(per_head.sum().item()) * sum(due)


class HostPipeline:
    """Decode steps fed from pinned host memory with the PCIe copies hidden:
    step i's H2D inputs and step i-1's D2H outputs run on a copy stream while
    the compute stream executes the step graph (double-buffered device
    staging, ordered by CUDA events).  Every step still moves its own inputs
    host->device and its outputs device->host."""

    def __init__(self, eng: DecodeEngine):
        self.eng = eng
        dev = eng.device
        self.copy = torch.cuda.Stream(dev)      # H2D of upcoming inputs
        self.copy_out = torch.cuda.Stream(dev)  # D2H of finished outputs (separate queue:
        self.main = torch.cuda.current_stream(dev)  # an H2D never waits behind a D2H)
        self.q = [torch.empty_like(eng.q) for _ in range(2)]
        self.k = [torch.empty_like(eng.k_new) for _ in range(2)]
        self.v = [torch.empty_like(eng.v_new) for _ in range(2)]
        self.o = [torch.empty_like(eng.out) for _ in range(2)]
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_used = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_used + self.ev_out:
            e.record(self.main)
        self.i = 0

    def submit(self, q_host, k_host, v_host, out_host) -> None:
        s = self.i % 2
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(self.ev_used[s])  # step i-2 consumed this staging set
            self.q[s].copy_(q_host, non_blocking=True)
            self.k[s].copy_(k_host, non_blocking=True)
            self.v[s].copy_(v_host, non_blocking=True)
            self.ev_in[s].record(self.copy)
        self.main.wait_event(self.ev_in[s])
        self.eng.q.copy_(self.q[s])
        self.eng.k_new.copy_(self.k[s])
        self.eng.v_new.copy_(self.v[s])
        self.eng.step()
        self.main.wait_event(self.ev_out[s])  # step i-2's outputs left this buffer
        self.o[s].copy_(self.eng.out)
        self.ev_used[s].record(self.main)
        with torch.cuda.stream(self.copy_out):
            self.copy_out.wait_event(self.ev_used[s])
            out_host.copy_(self.o[s], non_blocking=True)
            self.ev_out[s].record(self.copy_out)
        self.i += 1

    def drain(self) -> None:
        """Make the compute stream wait for every outstanding copy."""
        self.main.wait_stream(self.copy)
        self.main.wait_stream(self.copy_out)
