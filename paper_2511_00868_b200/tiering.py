"""Two-tier page placement — the reference's ``tierkv.tiering`` semantics
(tiering.py:42-184) with real data movement.

The slow tier is pinned host memory ``[B, L, H, N_cap, page]`` (same in-page
layout as the HBM pool); pages move with zero-copy UVA kernels
(fc_offload_pages: HBM -> host, fc_fetch_pages: host -> HBM over a copy list
produced by fc_rerank_recycle), on whatever stream the caller uses (a side
stream overlapped with decode, ordered by CUDA events).  The write-once
offload ledger, stable-only rule and capacity check follow the reference:
every full page of a stable head is written exactly once (tiering.py:99-157),
unstable heads never offload or reload (:146-148, :164-166).  The
latency/bandwidth cost model (tiering.py:29-39) is replaced by measurement.
"""

from __future__ import annotations

import numpy as np
import torch

from .config import HeadId
from .errors import AdmissionError, ConsistencyError
from .store import PAGE_SIZE, KVStore


def promoted_delta(old_topk, new_topk) -> tuple:
    """Pages entering the selection, i.e. the ones that need a reload (tiering.py:42-46)."""
    old = {int(p) for p in getattr(old_topk, "pages", old_topk)}
    new = {int(p) for p in getattr(new_topk, "pages", new_topk)}
    return tuple(sorted(new - old))


class TierStore:
    """Pinned-host slow tier + write-once ledger for one KVStore."""

    def __init__(self, store: KVStore, profile, capacity_bytes: int | None = None):
        self.store = store
        self.profile = profile
        self.page_bytes = store.page_bytes
        cap_pages = store.B * store.L * store.H * store.NCAP
        self.capacity_bytes = cap_pages * self.page_bytes if capacity_bytes is None else capacity_bytes
        # [B, L, H, N, 2, ps, d] in the pool's element type, pinned
        self.host = torch.empty((store.B, store.L, store.H, store.NCAP, 2, PAGE_SIZE, store.D),
                                dtype=store.dtype, pin_memory=True)
        self.slow_resident = torch.zeros((store.B, store.L, store.H, store.NCAP), dtype=torch.uint8,
                                         device=store.device)
        self._counts: dict = {}
        self.slow_bytes_used = 0
        self.stable = tuple(profile.stable)

    def _record(self, row: int, head: HeadId, pages) -> np.ndarray:
        # ledger: per (row, head) a count per logical page (numpy, so a
        # post-prefill offload of thousands of pages is one vector check)
        key = (row, HeadId(*head))
        counts = self._counts.get(key)
        if counts is None:
            counts = self._counts[key] = np.zeros(self.store.NCAP, dtype=np.uint8)
        pages = np.asarray(pages, dtype=np.int64).reshape(-1)
        if pages.size and (counts[pages].any() or np.bincount(pages, minlength=1).max() > 1):
            dup = next(int(p) for p in pages if counts[p] or (pages == p).sum() > 1)
            raise ConsistencyError(f"page {dup} of {head} offloaded twice for request row {row}")
        n_bytes = int(pages.size) * self.page_bytes
        if self.slow_bytes_used + n_bytes > self.capacity_bytes:
            self._refresh_usage()
        if self.slow_bytes_used + n_bytes > self.capacity_bytes:
            raise AdmissionError(f"slow tier capacity exceeded: {self.slow_bytes_used + n_bytes} "
                                 f"> {self.capacity_bytes}")
        counts[pages] = 1
        self.slow_bytes_used += n_bytes
        return pages

    def _offload(self, entries, max_ctas: int = 0) -> int:
        if len(entries) == 0:
            return 0
        t = torch.as_tensor(entries, dtype=torch.int32).reshape(-1, 4).to(self.store.device)
        self.store.offload_pages(self.host, t, max_ctas)
        r, l, h, p = t.long().unbind(1)
        self.slow_resident[r, l, h, p] = 1
        return t.shape[0] * self.page_bytes

    def offload_after_prefill(self, row: int, full_pages: int, max_ctas: int = 0) -> int:
        """One background copy of every full stable-head page (tiering.py:122-139);
        ``max_ctas`` bounds the SMs the copy occupies (0: the whole GPU)."""
        if full_pages < 0:
            raise ValueError("full_pages must be non-negative")
        for head in self.stable:
            c = self._counts.get((row, head))
            if c is not None and c.any():
                raise ConsistencyError(f"request row {row} already ran its post-prefill offload")
        for head in self.stable:
            self._record(row, head, np.arange(full_pages))
        if full_pages == 0 or not self.stable:
            return 0
        # the copy list (row, layer, head, page) built on the device
        dev = self.store.device
        if getattr(self, "_stable_dev", None) is None:
            self._stable_dev = torch.tensor([[h.layer, h.head] for h in self.stable], dtype=torch.int32,
                                            device=dev)
            mask = torch.zeros((self.store.L, self.store.H, 1), dtype=torch.bool)
            for h in self.stable:
                mask[h.layer, h.head] = True
            self._stable_mask = mask.to(dev)
        heads = self._stable_dev
        n = len(self.stable) * full_pages
        e = torch.empty((len(self.stable), full_pages, 4), dtype=torch.int32, device=dev)
        e[..., 0] = row
        e[..., 1] = heads[:, :1]
        e[..., 2] = heads[:, 1:]
        e[..., 3] = torch.arange(full_pages, dtype=torch.int32, device=dev)
        e = e.view(n, 4)
        self.store.offload_pages(self.host, e, max_ctas)
        # (a masked fill: advanced-index assignment would synchronise the stream)
        self.slow_resident[row, :, :, :full_pages].masked_fill_(self._stable_mask, 1)
        return n * self.page_bytes

    def incremental_offload(self, row: int, head: HeadId, page: int, *, page_full: bool = True) -> int:
        """Copy one page that just became full (tiering.py:141-157)."""
        head = HeadId(*head)
        if self.profile.is_unstable(head):
            raise ConsistencyError(f"{head} is unstable; its pages are never offloaded")
        if not page_full:
            raise ConsistencyError(f"page {page} is not full; offload refused")
        self._record(row, head, [page])
        return self._offload([row, head.layer, head.head, int(page)])

    def reload(self, layer: int, copies: torch.Tensor, n_copies: torch.Tensor) -> None:
        """Fetch promoted pages (copy list from fc_rerank_recycle) host -> HBM."""
        self.store.fetch_pages(layer, self.host, copies, n_copies)

    def release_row(self, row: int) -> None:
        """A finished request: its slow-tier pages are no longer needed (the
        ledger entries and the bytes they held are released; the row may host
        a new request, whose write-once ledger starts empty)."""
        for key in [k for k in self._counts if k[0] == row]:
            self.slow_bytes_used = max(0, self.slow_bytes_used - int(self._counts.pop(key).sum()) * self.page_bytes)
        self.slow_resident[row].zero_()

    def _refresh_usage(self) -> None:
        # pages filled during decode are offloaded inside the step graph
        # (fc_offload_filled sets slow_resident on the device; a second write
        # of a page raises FC_ERR_WRITE_TWICE there): the slow-tier bytes in
        # use are the device flags plus host-ledgered pages not flagged yet
        torch.cuda.current_stream(self.store.device).synchronize()
        flags = self.slow_resident.cpu().numpy()
        extra = 0
        for (row, head), c in self._counts.items():
            extra += int((c.astype(bool) & ~flags[row, head.layer, head.head].astype(bool)).sum())
        self.slow_bytes_used = (int(flags.sum()) + extra) * self.page_bytes

    def offload_counts(self, row: int, head: HeadId) -> dict:
        """Pages of (row, head) in the slow tier, each written once: the
        host-ledgered offloads (post-prefill, incremental) and the decode-time
        offloads recorded on the device (tiering.py:99-157)."""
        head = HeadId(*head)
        c = self._counts.get((row, head))
        dev = self.slow_resident[row, head.layer, head.head].cpu().numpy().astype(bool)
        if c is not None:
            dev |= c.astype(bool)
        return {int(p): 1 for p in np.flatnonzero(dev)}

    def slow_pages(self, row: int, head: HeadId) -> set:
        return set(self.offload_counts(row, head))


class ReloadStager:
    """Reload staging: the paper's transfer/compute overlap
    for the request itself.  ``leads`` steps before a rerank, every stable head
    is scored with that step's query into a separate PREDICTED selection
    (fc_score_select through a second store view) on a side stream; the pages
    it would promote that have a slow-tier copy are fetched host -> a staging
    area in HBM there (fc_stage_promoted) while decode continues.  At the
    rerank the real selection, recycle and copy list are computed as always;
    fc_fetch_pages_staged takes every staged page from HBM and only the
    mispredicted ones over the host link.  Results are identical with or
    without staging."""

    def __init__(self, store: KVStore, tier: TierStore, unstable: torch.Tensor, topk: int,
                 leads=(2,), capacity: int | None = None):
        st = self.store = store
        self.tier = tier
        self.topk = topk
        # predictions made this many steps before each rerank (each stages the
        # pages the earlier ones did not).  Default one, two steps ahead:
        # (2, 1) staged 80 % instead of 64 % of the promotions at config 3 but
        # the second prediction cost more than the misses it saved
        self.leads = tuple(sorted(set(int(x) for x in leads), reverse=True))[:4]
        self.lead = self.leads[0]
        self._pass = 0
        dev = st.device
        n_stable = int((unstable == 0).sum().item())
        if capacity is None:  # every stable head replacing its whole selection
            capacity = max(1, min(st.B * n_stable * topk, 1 << 17))
        self.capacity = capacity
        self.unstable = unstable
        self.stable_mask = (unstable == 0).to(torch.uint8).contiguous()
        self.pred_sel = torch.zeros_like(st.sel)
        self.pred_n = torch.zeros_like(st.n_sel)
        # every layer scored as one layer of L*H heads (KVStore.score_select_all_layers_into)
        self.pred_scores = torch.full((st.B * st.L * st.H, st.NCAP), float("-inf"), dtype=torch.float32,
                                      device=dev)
        self.pred_counters = torch.zeros(st.B * st.L * st.H, dtype=torch.int32, device=dev)
        self.q_bl = None
        self.staged_map = torch.full(tuple(st.table.shape), -1, dtype=torch.int32, device=dev)
        self.stage_list = torch.zeros((capacity, 2), dtype=torch.int32, device=dev)
        self.stage_count = torch.zeros(9, dtype=torch.int32, device=dev)  # [taken, (first, end) x 4 passes]
        self.staging = torch.empty((capacity, 2, PAGE_SIZE, st.D), dtype=st.dtype, device=dev)
        self.hits = torch.zeros(1, dtype=torch.int64, device=dev)
        self._hits32 = torch.zeros(1, dtype=torch.int32, device=dev)
        self.staged_pages = torch.zeros(1, dtype=torch.int64, device=dev)
        # low priority: the host-link copies yield SMs to decode
        self.stream = torch.cuda.Stream(dev, priority=0)
        self.ev_input = torch.cuda.Event()
        self.ev_staged = torch.cuda.Event()
        self.pending = False

    def predict(self, q: torch.Tensor, batch: int, layers) -> None:
        """Predict and stage from the query ``q`` [L, B, Hq, d] of the step
        that just ran (copied first: the caller may overwrite it)."""
        # the prediction runs on the current stream (scoring kernels fill every
        # SM: on a side stream they would stall the next step's launches); only
        # the host-link copies go to the side stream, on a few SMs
        main = torch.cuda.current_stream(self.store.device)
        if self.q_bl is None:
            self.q_bl = torch.empty((q.shape[1], q.shape[0]) + tuple(q.shape[2:]), dtype=q.dtype, device=q.device)
        self.q_bl.copy_(q.transpose(0, 1))  # [B, L, Hq, d]: the all-layers view's query layout
        self.store.score_select_all_layers_into(self.q_bl, self.stable_mask, self.topk, batch, self.pred_sel,
                                                self.pred_n, self.pred_scores, self.pred_counters)
        k = self._pass
        self.store.stage_plan(self.pred_sel, self.pred_n, self.unstable, self.tier.slow_resident,
                              self.staged_map, self.stage_list, self.stage_count, self.capacity, batch, k)
        self.ev_input.record(main)
        with torch.cuda.stream(self.stream):
            self.stream.wait_event(self.ev_input)
            self.store.stage_fetch(self.tier.host, self.stage_list, self.stage_count, self.staging, k)
            self.ev_staged.record(self.stream)
        self._pass = min(k + 1, 3)
        self.pending = True

    def wait(self) -> None:
        """Order the current stream after the staging copies (before a rerank)."""
        if self.pending:
            torch.cuda.current_stream(self.store.device).wait_event(self.ev_staged)
            self.pending = False

    def fetch(self, layer: int, copies: torch.Tensor, n_copies: torch.Tensor) -> None:
        self.store.fetch_pages_staged(layer, self.tier.host, copies, n_copies, self.staged_map, self.staging,
                                      self._hits32)

    def finish_rerank(self) -> None:
        """After the rerank's fetches (same stream): count hits, clear the map."""
        self.hits.add_(self._hits32.long())
        self._hits32.zero_()
        self.staged_pages.add_(self.stage_count[0].clamp(max=self.capacity).long())
        self.store.stage_clear(self.staged_map, self.stage_list, self.stage_count, self.capacity)

    def forget_row(self, row: int) -> None:
        """A retired row: drop its staged pages before the row can host a new
        request (the staging map is indexed by (row, layer, head, page); a stale
        entry would hand the old request's page to the new one at its first
        rerank).  The current stream first waits for the staging copies, so no
        copy still reads the old request's host slots when the new request's
        offload overwrites them."""
        if self.pending:
            torch.cuda.current_stream(self.store.device).wait_event(self.ev_staged)
        self.staged_map[row].fill_(-1)

    def rerank_launched(self) -> None:
        """Host bookkeeping after a rerank step was launched (the step graph
        replays finish_rerank's device work): the next prediction is pass 0."""
        self._pass = 0
