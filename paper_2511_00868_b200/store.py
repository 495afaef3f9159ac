"""KVStore: the GPU-resident, batched state of the FlexiCache hot path.

One ``KVStore`` holds, for ``batch_cap`` request rows × L layers × H KV heads:

* the physical KV pool ``[n_blocks, 2, ps, d]`` (block 0 = null block) —
  ``PhysicalPool`` (blocktable.py:28-94) with its LIFO free list kept on the
  device (``free_stack``/``free_top``);
* the dense logical→physical table ``[B, L, H, N_cap]`` int32 —
  ``BlockTable`` (blocktable.py:109-440);
* the per-page key min/max summaries ``[B, L, H, N_cap, 2, d]`` —
  ``MinMaxCache`` (scoring.py:114-139);
* the current page selection per head ``[B, L, H, sel_cap]`` + count —
  ``TopKSet`` (scoring.py:142-161);
* ``seq_len[B]``, the decode step counter and a sticky device error word.

All buffers are torch tensors; the C-ABI library (``_lib``) only receives
their device pointers.  Every method is asynchronous on the current CUDA
stream except ``check_errors`` and the host readbacks.
"""

from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _lib
from .errors import ConsistencyError, PoolExhausted

PAGE_SIZE = 16
_DTYPES = {torch.bfloat16: _lib.FC_BF16, torch.float32: _lib.FC_F32}


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class KVStore:
    def __init__(self, *, batch_cap: int, layers: int, kv_heads: int, group: int,
                 head_dim: int, pages_cap: int, n_blocks: int, sel_cap: int,
                 dtype: torch.dtype = torch.bfloat16, device="cuda"):
        if dtype not in _DTYPES:
            raise ValueError("dtype must be torch.bfloat16 or torch.float32")
        if n_blocks < 2:
            raise ValueError("pool needs at least one real block beyond the null block")
        self.lib = _lib.load()
        self.device = torch.device(device)
        if self.device.type != "cuda" or not torch.cuda.is_available():
            raise RuntimeError("KVStore needs a CUDA device (B200, sm_100a); no CPU fallback")
        self.B, self.L, self.H, self.G = batch_cap, layers, kv_heads, group
        self.D, self.PS, self.NCAP, self.SELCAP = head_dim, PAGE_SIZE, pages_cap, sel_cap
        self.dtype, self.n_blocks = dtype, n_blocks
        dev = self.device
        self.kv_pool = torch.zeros((n_blocks, 2, PAGE_SIZE, head_dim), dtype=dtype, device=dev)
        self.summaries = torch.zeros((batch_cap, layers, kv_heads, pages_cap, 2, head_dim),
                                     dtype=dtype, device=dev)
        self.table = torch.zeros((batch_cap, layers, kv_heads, pages_cap), dtype=torch.int32, device=dev)
        self.seq_len = torch.zeros(batch_cap, dtype=torch.int32, device=dev)
        self.sel = torch.zeros((batch_cap, layers, kv_heads, sel_cap), dtype=torch.int32, device=dev)
        self.n_sel = torch.zeros((batch_cap, layers, kv_heads), dtype=torch.int32, device=dev)
        # fresh pool pops 1, 2, 3, ... (blocktable.py:38-39)
        self.free_stack = torch.arange(n_blocks - 1, 0, -1, dtype=torch.int32, device=dev)
        self.free_stack = torch.cat([self.free_stack, torch.zeros(1, dtype=torch.int32, device=dev)])
        self.free_top = torch.tensor([n_blocks - 1], dtype=torch.int32, device=dev)
        self.step = torch.ones(1, dtype=torch.int32, device=dev)
        self.error_word = torch.zeros(1, dtype=torch.int32, device=dev)
        # per-request decode state: row b's own step t_b = step + row_phase[b]
        # (simulator.py:437-439) and its reload-pause mode (FC_HOLD_*)
        self.row_phase = torch.zeros(batch_cap, dtype=torch.int32, device=dev)
        self.row_hold = torch.zeros(batch_cap, dtype=torch.uint8, device=dev)
        # device scoring counters (FC_STAT_*: Metrics, simulator.py:87-131)
        self.stats = torch.zeros(_lib.FC_STATS_N, dtype=torch.int64, device=dev)
        self._c = _lib.FcStore(
            batch_cap, layers, kv_heads, group, head_dim, PAGE_SIZE, pages_cap, sel_cap,
            _DTYPES[dtype], n_blocks,
            self.kv_pool.data_ptr(), self.summaries.data_ptr(), self.table.data_ptr(),
            self.seq_len.data_ptr(), self.sel.data_ptr(), self.n_sel.data_ptr(),
            self.free_stack.data_ptr(), self.free_top.data_ptr(), self.step.data_ptr(),
            self.error_word.data_ptr(), self.row_phase.data_ptr(), self.row_hold.data_ptr(),
            self.stats.data_ptr())
        # the descriptor kernels see: with the per-request state only while some
        # row is out of phase or held (``per_row``); in phase, every kernel
        # skips those loads (they sat on the attention prologue's dependent
        # chain: +0.7 us per launch at config 2)
        self._c_phase = self._c
        self._c_flat = _lib.FcStore.from_buffer_copy(self._c)
        self._c_flat.row_phase = None
        self._c_flat.row_hold = None
        self.per_row = False
        # fc_score_attend_balanced_ws: the scored heads' attention cut into
        # chunks that idle CTAs claim (FC_BAL_CHUNKS per head).  Off by
        # default (FC_BAL_HELPERS=1: on): measured slower at config 2 with
        # the spread mask (9.6k vs 12.8k tokens/s)
        self.balanced_helpers = os.environ.get("FC_BAL_HELPERS", "0") == "1"
        # the same store without the counters: selections that are not
        # scheduled score evaluations (initial selection, reload prediction)
        self._c_quiet = _lib.FcStore.from_buffer_copy(self._c)
        self._c_quiet.stats = None
        self.cptr_quiet = ctypes.addressof(self._c_quiet)
        # scoring workspace: scores [B*H, N_cap] fp32 + per-head counters
        self.scores = torch.full((batch_cap * kv_heads, pages_cap), float("-inf"),
                                 dtype=torch.float32, device=dev)
        self.score_counters = torch.zeros(batch_cap * kv_heads, dtype=torch.int32, device=dev)
        self._attn_ws = torch.zeros(0, dtype=torch.uint8, device=dev)
        self._rerank_ws = None
        self._run_ws = torch.zeros(0, dtype=torch.uint8, device=dev)

    # -- misc ------------------------------------------------------------------

    @property
    def cptr(self) -> int:
        return ctypes.addressof(self._c_phase if self.per_row else self._c_flat)

    @property
    def page_bytes(self) -> int:
        return 2 * PAGE_SIZE * self.D * self.kv_pool.element_size()

    def stream(self) -> int:
        return _stream(self.device)

    def check_errors(self) -> None:
        """Synchronise and raise the reference exception for any sticky
        device error bit (then clear it)."""
        bits = int(self.error_word.item()) & 0xFFFFFFFF
        if not bits:
            return
        self.error_word.zero_()
        if bits & _lib.FC_ERR_POOL_EXHAUSTED:
            raise PoolExhausted(f"fast pool exhausted ({self.n_blocks - 1} blocks)")
        if bits & _lib.FC_ERR_WRITE_TWICE:
            raise ConsistencyError("page offloaded twice (write-once ledger, tiering.py:105-110)")
        if bits & (_lib.FC_ERR_NULL_READ | _lib.FC_ERR_DOUBLE_EVICT):
            raise ConsistencyError(
                "residency violation: read of the null block / double eviction "
                f"(device error bits {bits:#x})")
        if bits & _lib.FC_ERR_NULL_WRITE:
            raise ConsistencyError("append into a page with no physical block")
        if bits & _lib.FC_ERR_TRACE_SHORT:
            raise ValueError("trace capture: a selection shorter than K (candidate pool <= K)")
        raise ValueError(f"capacity exceeded (device error bits {bits:#x})")

    def free_count(self) -> int:
        return int(self.free_top.item())

    # -- allocation / steps ------------------------------------------------------

    def alloc_pages(self, row: int, first_page: int, n_pages: int) -> None:
        _lib.check(self.lib.fc_alloc_pages(self.cptr, row, first_page, n_pages, self.stream()),
                   "fc_alloc_pages")

    def free_row(self, row: int) -> None:
        """Release every page of request row ``row`` and mark it free
        (seq_len = -1: skipped by every kernel) — fc_free_row."""
        _lib.check(self.lib.fc_free_row(self.cptr, row, self.stream()), "fc_free_row")

    def row_view(self, row: int) -> int:
        """An fc_store of the single request row ``row`` (batch_cap 1, the
        per-row buffers offset to it; pool, free list and step shared): a
        call through it touches that row only (e.g. the initial selection of
        a request admitted mid-stream)."""
        views = self.__dict__.setdefault("_row_views", {})
        if row not in views:
            if not 0 <= row < self.B:
                raise ValueError("row out of range")
            c = _lib.FcStore.from_buffer_copy(self._c)
            c.batch_cap = 1
            c.table = self.table[row].data_ptr()
            c.summaries = self.summaries[row].data_ptr()
            c.seq_len = self.seq_len[row:row + 1].data_ptr()
            c.sel = self.sel[row].data_ptr()
            c.n_sel = self.n_sel[row].data_ptr()
            c.row_phase = self.row_phase[row:row + 1].data_ptr()
            c.row_hold = self.row_hold[row:row + 1].data_ptr()
            c.stats = None  # (initial selections: not scheduled evaluations)
            views[row] = c
        return ctypes.addressof(views[row])

    def score_select_row(self, row: int, layer: int, q_row: torch.Tensor, unstable: torch.Tensor, period: int,
                         topk: int, *, force_due: bool = True, extra_tokens: int = 1) -> None:
        """fc_score_select of one request row (q_row: [Hq, d] of that row)."""
        _lib.check(self.lib.fc_score_select(
            self.row_view(row), layer, q_row.data_ptr(), unstable.data_ptr(), period, int(force_due), topk,
            extra_tokens, 0, self.scores.data_ptr(), self.score_counters.data_ptr(), 1, self.stream()),
            "fc_score_select")

    def step_advance(self, batch: int, unstable: torch.Tensor | None = None, period: int = 1) -> None:
        """fc_step_advance; with ``unstable`` / ``period`` also count the
        step's skipped layers into ``stats`` (fc_step_advance_counted)."""
        if unstable is None:
            _lib.check(self.lib.fc_step_advance(self.cptr, batch, self.stream()), "fc_step_advance")
        else:
            _lib.check(self.lib.fc_step_advance_counted(self.cptr, batch, unstable.data_ptr(), period,
                                                        self.stream()), "fc_step_advance_counted")

    def scoring_stats(self) -> dict:
        """The device counters (synchronising read): heads scored, the naive
        count (every head of every decoding row every step), (row, layer)
        pairs with no due head, row-steps held for a reload."""
        v = self.stats.tolist()
        return {"score_evals": v[_lib.FC_STAT_SCORE_EVALS],
                "score_evals_naive": v[_lib.FC_STAT_SCORE_EVALS_NAIVE],
                "layer_scoring_skips": v[_lib.FC_STAT_LAYER_SKIPS],
                "held_row_steps": v[_lib.FC_STAT_HELD_ROW_STEPS]}

    def evict_pages(self, pages: torch.Tensor) -> None:
        """pages: int32 [n, 4] (row, layer, head, logical) on the device."""
        pages = pages.to(self.device, torch.int32).contiguous()
        _lib.check(self.lib.fc_evict_pages(self.cptr, pages.data_ptr(), pages.shape[0], self.stream()),
                   "fc_evict_pages")

    # -- (1) KV writes -------------------------------------------------------------

    def prefill(self, row: int, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        """k, v: [H, T, d] in the store dtype, on the device."""
        k = k.to(self.device, self.dtype).contiguous()
        v = v.to(self.device, self.dtype).contiguous()
        if k.shape != v.shape or k.dim() != 3 or k.shape[0] != self.H or k.shape[2] != self.D:
            raise ValueError("k and v must both be [H, T, d]")
        _lib.check(self.lib.fc_kv_prefill(self.cptr, row, layer, k.data_ptr(), v.data_ptr(),
                                          k.shape[1], self.stream()), "fc_kv_prefill")

    def append(self, layer: int, k_new: torch.Tensor, v_new: torch.Tensor, batch: int) -> None:
        """k_new, v_new: [batch, H, d] contiguous in the store dtype."""
        _lib.check(self.lib.fc_kv_append(self.cptr, layer, k_new.data_ptr(), v_new.data_ptr(),
                                         batch, self.stream()), "fc_kv_append")

    def gather(self, row: int, layer: int, head: int, n_pages: int):
        """Logical K/V [n_pages*ps, d] of one head (un-swizzled readback)."""
        k = torch.empty((n_pages * PAGE_SIZE, self.D), dtype=self.dtype, device=self.device)
        v = torch.empty_like(k)
        _lib.check(self.lib.fc_kv_gather(self.cptr, row, layer, head, n_pages, k.data_ptr(),
                                         v.data_ptr(), self.stream()), "fc_kv_gather")
        return k, v

    # -- (2) scoring / selection -----------------------------------------------------

    def score_select(self, layer: int, q: torch.Tensor, unstable: torch.Tensor, period: int,
                     topk: int, batch: int, *, force_due: bool = False, extra_tokens: int = 1,
                     kv_prefetch: bool = False, counted: bool = True) -> None:
        _lib.check(self.lib.fc_score_select(
            self.cptr if counted else self.cptr_quiet, layer, q.data_ptr(), unstable.data_ptr(), period, int(force_due), topk,
            extra_tokens, int(kv_prefetch), self.scores.data_ptr(), self.score_counters.data_ptr(),
            batch, self.stream()), "fc_score_select")

    def score_attend_supported(self, batch: int) -> int:
        """CTAs per head fc_score_attend uses for this batch (0: unsupported)."""
        return int(self.lib.fc_score_attend_supported(self.cptr, batch))

    def score_attend(self, layer: int, q: torch.Tensor, unstable: torch.Tensor, period: int, topk: int,
                     out: torch.Tensor, batch: int, *, force_due: bool = False, extra_tokens: int = 1,
                     kv_prefetch: bool = False, k_new: torch.Tensor | None = None,
                     v_new: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                     scale: float | None = None, attend_appended: bool = False,
                     cta_map: torch.Tensor | None = None, cluster: int = 0) -> None:
        """fc_score_attend: score_select then sparse_decode of one layer, one
        CTA per head (same results as the two calls); with ``cta_map`` /
        ``cluster`` fc_score_attend_map (mixed clusters, mixed_cluster_map)."""
        scale = 1.0 / math.sqrt(self.D) if scale is None else scale
        if cta_map is not None:
            _lib.check(self.lib.fc_score_attend_map(
                self.cptr, layer, q.data_ptr(), unstable.data_ptr(), period, int(force_due), topk, extra_tokens,
                int(kv_prefetch), self.scores.data_ptr(), _ptr(k_new), _ptr(v_new), out.data_ptr(), _ptr(lse),
                scale, int(attend_appended), batch, cta_map.data_ptr(), cta_map.numel(), cluster,
                self.stream()), "fc_score_attend_map")
            return
        _lib.check(self.lib.fc_score_attend(
            self.cptr, layer, q.data_ptr(), unstable.data_ptr(), period, int(force_due), topk, extra_tokens,
            int(kv_prefetch), self.scores.data_ptr(), _ptr(k_new), _ptr(v_new), out.data_ptr(), _ptr(lse),
            scale, int(attend_appended), batch, self.stream()), "fc_score_attend")

    def score_attend_balanced_supported(self, batch: int) -> int:
        """Grid of fc_score_attend_balanced for this batch (0: unsupported)."""
        cache = self.__dict__.setdefault("_bal_grid", {})
        if batch not in cache:
            cache[batch] = int(self.lib.fc_score_attend_balanced_supported(self.cptr, batch))
        return cache[batch]

    def score_attend_balanced(self, layer: int, q: torch.Tensor, unstable: torch.Tensor, period: int, topk: int,
                              out: torch.Tensor, batch: int, *, force_due: bool = False, extra_tokens: int = 1,
                              kv_prefetch: bool = False, k_new: torch.Tensor | None = None,
                              v_new: torch.Tensor | None = None, lse: torch.Tensor | None = None,
                              scale: float | None = None, attend_appended: bool = False) -> None:
        """fc_score_attend_balanced: the due heads' scoring spread over every
        SM, then per head selection and attention (same results as
        fc_score_select's balanced kernel followed by fc_sparse_decode)."""
        scale = 1.0 / math.sqrt(self.D) if scale is None else scale
        ws = None
        if self.balanced_helpers:
            need = int(self.lib.fc_score_attend_balanced_workspace_size(self.cptr, batch))
            ws = self.__dict__.get("_bal_ws")
            if ws is None or ws.numel() < need:
                ws = self._bal_ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        _lib.check(self.lib.fc_score_attend_balanced_ws(
            self.cptr, layer, q.data_ptr(), unstable.data_ptr(), period, int(force_due), topk, extra_tokens,
            int(kv_prefetch), self.scores.data_ptr(), self.score_counters.data_ptr(), _ptr(k_new), _ptr(v_new),
            out.data_ptr(), _ptr(lse), scale, int(attend_appended), batch, _ptr(ws), 0 if ws is None else ws.numel(),
            self.stream()), "fc_score_attend_balanced_ws")

    def score_attend_map_fits(self, n_ctas: int, cluster: int) -> bool:
        cache = self.__dict__.setdefault("_map_fits", {})
        if (n_ctas, cluster) not in cache:
            cache[(n_ctas, cluster)] = bool(self.lib.fc_score_attend_map_fits(self.cptr, n_ctas, cluster))
        return cache[(n_ctas, cluster)]

    def mixed_cluster_map(self, batch: int, scored_heads, n_pages: int, topk_pages: int, *,
                          sms: int | None = None, bw_sm_gbs: float = 90.0, bw_gbs: float = 6000.0):
        """A CTA map for fc_score_attend_map that balances a launch in which
        only ``scored_heads`` (kv-head indices of the layer, every row) are
        scored: each scored head gets a cluster of S CTAs, the other heads
        one CTA each, S CTAs to a cluster.  Chosen by a bandwidth model (each
        CTA streams at most ``bw_sm_gbs``, the launch at most ``bw_gbs``);
        None when the uniform launch (fc_score_attend) models as fast or the
        mixed grid does not fit.  Returns (map [n_ctas] int32 on the device,
        cluster)."""
        if sms is None:
            if not hasattr(self, "_sms"):
                self._sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            sms = self._sms
        scored = sorted(set(int(h) for h in scored_heads))
        if not scored or len(scored) == self.H:  # nothing to balance: the uniform launch
            return None
        n_s = batch * len(scored)
        n_o = batch * self.H - n_s
        att = min(n_pages, topk_pages + 2) * self.page_bytes
        summ = n_pages * 2 * self.D * self.kv_pool.element_size()

        def est(per_cta):
            total = n_s * (summ + att) + n_o * att
            return max(per_cta / (bw_sm_gbs * 1e3), total / (bw_gbs * 1e3))  # us

        su = self.score_attend_supported(batch)
        if su < 1:
            return None
        best = None
        for S in range(2, 17):
            clusters = n_s + (n_o + S - 1) // S
            if clusters * S > sms or not self.score_attend_map_fits(clusters * S, S):
                continue
            per = max((summ + att) / S, att if n_o else 0)
            t = (est(per), per)  # ties: the smaller per-CTA share
            if best is None or t < best[0]:
                best = (t, S)
        if best is None or best[0][0] >= 0.9 * est((summ + att) / su):
            return None
        S = best[1]
        m = []
        others = []
        for b in range(batch):
            for h in range(self.H):
                bh = b * self.H + h
                if h in scored:
                    m += [bh] * S
                else:
                    others.append(bh | (1 << 30))
        others += [-1] * (-len(others) % S)
        m += others
        return torch.tensor(m, dtype=torch.int32, device=self.device), S

    def cluster_plan(self, batch: int, n_scored: int, n_pages: int, topk_pages: int, *,
                     sms: int | None = None, bw_sm_gbs: float = 90.0, bw_gbs: float = 6000.0,
                     select_us: float = 0.0):
        """The cluster size S for a launch in which ``n_scored`` of the
        batch's (row, head) pairs are scored (any pairs: e.g. every head of
        the rows at their rerank boundary), by the bandwidth model of
        ``mixed_cluster_map``: (S, CTAs) or None when the uniform launch models
        as fast or no one-wave grid fits."""
        if sms is None:
            if not hasattr(self, "_sms"):
                self._sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            sms = self._sms
        n_s, n_o = n_scored, batch * self.H - n_scored
        if n_s <= 0 or n_o <= 0:
            return None
        att = min(n_pages, topk_pages + 2) * self.page_bytes
        summ = n_pages * 2 * self.D * self.kv_pool.element_size()

        def est(scored_cta, other_cta):
            # a scored head's CTAs stream their share, then wait for the selection
            total = n_s * (summ + att) + n_o * att
            t_cta = max(scored_cta / (bw_sm_gbs * 1e3) + select_us, other_cta / (bw_sm_gbs * 1e3))
            return max(t_cta, total / (bw_gbs * 1e3))  # us

        su = self.score_attend_supported(batch)
        if su < 1:
            return None
        best = None
        for S in (2, 4, 8, 16):  # (clusters of 3 leave GPC SMs unused: a second wave, partial_probe.py)
            n_ctas = (n_s + (n_o + S - 1) // S) * S
            if n_ctas > sms or not self.score_attend_map_fits(n_ctas, S):
                continue
            t = (est((summ + att) / S, att), S)
            if best is None or t < best[0]:
                best = (t, S, n_ctas)
        if best is None or best[0][0] >= 0.9 * est((summ + att) / su, att / su):
            return None
        return best[1], best[2]

    def cluster_map_pairs(self, batch: int, scored, S: int, n_ctas: int) -> torch.Tensor:
        """Host map for fc_score_attend_map: each (row, head) in ``scored`` a
        cluster of S CTAs, every other head one CTA (bit 30), S to a cluster;
        padded with idle CTAs (-1) to ``n_ctas``."""
        scored = set(scored)
        n_all = batch * self.H
        while scored and len(scored) * S + -(-(n_all - len(scored)) // S) * S > n_ctas:
            scored.discard(max(scored))  # too many for the grid: the rest attend (and score) alone
        m, others = [], []
        for b in range(batch):
            for h in range(self.H):
                bh = b * self.H + h
                if (b, h) in scored:
                    m += [bh] * S
                else:
                    others.append(bh | (1 << 30))
        others += [-1] * (-len(others) % S)
        m += others
        if len(m) > n_ctas:
            raise ValueError(f"map needs {len(m)} CTAs > {n_ctas}")
        m += [-1] * (n_ctas - len(m))
        return torch.tensor(m, dtype=torch.int32)

    def score_pages(self, layer: int, q: torch.Tensor, batch: int, *, extra_tokens: int = 0) -> None:
        _lib.check(self.lib.fc_score_pages(self.cptr, layer, q.data_ptr(), extra_tokens,
                                           self.scores.data_ptr(), batch, self.stream()),
                   "fc_score_pages")

    # -- (3) attention -------------------------------------------------------------

    def attn_workspace(self, batch: int, max_pages: int, n_ctas: int = 0) -> torch.Tensor:
        need = self.lib.fc_sparse_decode_workspace_size(self.cptr, batch, max_pages, n_ctas)
        if self._attn_ws.numel() < need:
            self._attn_ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._attn_ws

    def sparse_decode(self, layer: int, q: torch.Tensor, out: torch.Tensor, batch: int, *,
                      max_pages: int, n_ctas: int = 0, lse: torch.Tensor | None = None,
                      scale: float | None = None, extra_tokens: int = 1,
                      attend_appended: bool = True, k_new: torch.Tensor | None = None,
                      v_new: torch.Tensor | None = None, kv_prefetch: bool = False,
                      early_unstable: torch.Tensor | None = None, early_period: int = 1) -> None:
        """Split-K paged attention; with k_new/v_new the decode append is fused.
        ``early_unstable`` (the [L, H] flags the preceding score_select used,
        with its period): heads it does not select this step start without
        waiting for it."""
        ws = self.attn_workspace(batch, max_pages, n_ctas)
        scale = 1.0 / math.sqrt(self.D) if scale is None else scale
        _lib.check(self.lib.fc_sparse_decode(
            self.cptr, layer, q.data_ptr(), _ptr(k_new), _ptr(v_new), out.data_ptr(), _ptr(lse),
            scale, extra_tokens, int(attend_appended), int(kv_prefetch), _ptr(early_unstable),
            early_period, max_pages, n_ctas, ws.data_ptr(),
            ws.numel(), batch, self.stream()), "fc_sparse_decode")

    def run_supported(self, batch: int, max_pages: int) -> bool:
        """Whether the persistent multi-layer kernel fits this geometry."""
        return bool(self.lib.fc_sparse_decode_layers_supported(self.cptr, batch, max_pages))

    def run_split(self, batch: int, max_pages: int) -> int:
        """CTAs per head of the per-head persistent kernel (0: warp-balanced)."""
        return int(self.lib.fc_sparse_decode_layers_split(self.cptr, batch, max_pages))

    def sparse_decode_layers(self, layer: int, n_layers: int, q: torch.Tensor, out: torch.Tensor,
                             batch: int, *, max_pages: int, lse: torch.Tensor | None = None,
                             scale: float | None = None, extra_tokens: int = 1,
                             attend_appended: bool = True, k_new: torch.Tensor | None = None,
                             v_new: torch.Tensor | None = None, first_dep: bool = True) -> None:
        """fc_sparse_decode_layers: the layers [layer, layer + n_layers) in one
        persistent launch.  q/out (and k_new/v_new, lse) are per-layer stacks
        ([n_layers, ...], dim 0 = layer); same per-(layer, head) semantics as
        sparse_decode."""
        need = self.lib.fc_sparse_decode_layers_workspace_size(self.cptr, batch, max_pages)
        if self._run_ws.numel() < need:
            self._run_ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        scale = 1.0 / math.sqrt(self.D) if scale is None else scale
        st = (lambda t: t.stride(0) if (t is not None and t.dim() > 0 and n_layers > 1) else 0)
        _lib.check(self.lib.fc_sparse_decode_layers(
            self.cptr, layer, n_layers, q.data_ptr(), st(q), _ptr(k_new), _ptr(v_new), st(k_new),
            out.data_ptr(), st(out), _ptr(lse), st(lse), scale, extra_tokens, int(attend_appended),
            int(first_dep), max_pages, self._run_ws.data_ptr(), self._run_ws.numel(), batch,
            self.stream()), "fc_sparse_decode_layers")

    # -- (4) rerank / tiers ------------------------------------------------------------

    def rerank_workspace(self) -> torch.Tensor:
        if self._rerank_ws is None:
            n = self.lib.fc_rerank_workspace_size(self.cptr)
            self._rerank_ws = torch.zeros(n, dtype=torch.uint8, device=self.device)
        return self._rerank_ws

    def rerank_recycle(self, layer: int, old_sel: torch.Tensor, n_old: torch.Tensor,
                       unstable: torch.Tensor, period: int, copies: torch.Tensor,
                       n_copies: torch.Tensor, batch: int, *, force_due: bool = False,
                       old_has_tail: bool = True, extra_tokens: int = 1,
                       slow_resident: torch.Tensor | None = None,
                       row_skip: torch.Tensor | None = None) -> None:
        ws = self.rerank_workspace()
        _lib.check(self.lib.fc_rerank_recycle_rows(
            self.cptr, layer, old_sel.data_ptr(), n_old.data_ptr(), unstable.data_ptr(), period,
            int(force_due), int(old_has_tail), extra_tokens, _ptr(slow_resident), _ptr(row_skip),
            copies.data_ptr(), copies.shape[0], n_copies.data_ptr(), ws.data_ptr(), batch,
            self.stream()), "fc_rerank_recycle_rows")

    def rerank_recycle_all_layers(self, old_sel: torch.Tensor, n_old: torch.Tensor, unstable: torch.Tensor,
                                  period: int, copies: torch.Tensor, n_copies: torch.Tensor, batch: int, *,
                                  extra_tokens: int = 1, slow_resident: torch.Tensor | None = None,
                                  row_skip: torch.Tensor | None = None) -> None:
        """fc_rerank_recycle_rows of EVERY layer in one launch, through the
        view of the L layers as one layer of L*H heads: old_sel / n_old in
        the store's own [B, L, H, ...] layout, one copy list (row, l*H + h,
        page, block) for fetch_pages_all_layers."""
        view = self._all_layers_view(self.sel, self.n_sel)
        if getattr(self, "_rerank_ws_all", None) is None:
            n = self.lib.fc_rerank_workspace_size(view)
            self._rerank_ws_all = torch.zeros(n, dtype=torch.uint8, device=self.device)
        ws = self._rerank_ws_all
        _lib.check(self.lib.fc_rerank_recycle_rows(
            view, 0, old_sel.data_ptr(), n_old.data_ptr(), unstable.data_ptr(), period, 0, 0, extra_tokens,
            _ptr(slow_resident), _ptr(row_skip), copies.data_ptr(), copies.shape[0], n_copies.data_ptr(),
            ws.data_ptr(), batch, self.stream()), "fc_rerank_recycle_rows")

    def fetch_pages_all_layers(self, host_pages: torch.Tensor, copies: torch.Tensor, n_copies: torch.Tensor,
                               max_ctas: int = 0, row: int = -1) -> None:
        """fc_fetch_pages_ctas of a copy list from rerank_recycle_all_layers
        (the entries of request row ``row`` only, -1: all)."""
        _lib.check(self.lib.fc_fetch_pages_ctas(self._all_layers_view(self.sel, self.n_sel), 0, host_pages.data_ptr(),
                                                copies.data_ptr(), n_copies.data_ptr(), copies.shape[0], row,
                                                max_ctas, self.stream()), "fc_fetch_pages_ctas")

    def trace_capture(self, trace_sel: torch.Tensor, trace_pool: torch.Tensor, step_base: int,
                      topk: int, batch: int, extra_tokens: int = 0) -> None:
        """Record every head's top-K selection into trace slot
        (device step - step_base) — fc_trace_capture."""
        _lib.check(self.lib.fc_trace_capture(self.cptr, trace_sel.data_ptr(), trace_pool.data_ptr(),
                                             step_base, trace_sel.shape[1], topk, extra_tokens, batch,
                                             self.stream()), "fc_trace_capture")

    def _view_with_sel(self, sel: torch.Tensor, n_sel: torch.Tensor) -> int:
        """An fc_store struct identical to this store's but whose selection
        buffers are ``sel`` / ``n_sel`` (same shapes): scoring through it
        writes a separate (e.g. predicted) selection."""
        key = (sel.data_ptr(), n_sel.data_ptr())
        views = self.__dict__.setdefault("_sel_views", {})
        if key not in views:
            if sel.shape != self.sel.shape or n_sel.shape != self.n_sel.shape:
                raise ValueError("selection buffers must match the store's sel / n_sel shapes")
            c = _lib.FcStore.from_buffer_copy(self._c_quiet)
            c.sel, c.n_sel = sel.data_ptr(), n_sel.data_ptr()
            views[key] = (c, (sel, n_sel))
        return ctypes.addressof(views[key][0])

    def _all_layers_view(self, sel: torch.Tensor, n_sel: torch.Tensor) -> int:
        """An fc_store view of every layer as ONE layer of L*H heads (flat
        head index (b*L + l)*H + h is unchanged, so table, summaries and the
        selection buffers are shared as they are) with the selection buffers
        replaced: one scoring launch covers all layers."""
        key = ("all", sel.data_ptr(), n_sel.data_ptr())
        views = self.__dict__.setdefault("_sel_views", {})
        if key not in views:
            if sel.shape != self.sel.shape or n_sel.shape != self.n_sel.shape:
                raise ValueError("selection buffers must match the store's sel / n_sel shapes")
            c = _lib.FcStore.from_buffer_copy(self._c_quiet)
            c.layers, c.kv_heads = 1, self.L * self.H
            c.sel, c.n_sel = sel.data_ptr(), n_sel.data_ptr()
            views[key] = (c, (sel, n_sel))
        return ctypes.addressof(views[key][0])

    def score_select_all_layers_into(self, q_bl: torch.Tensor, due_mask: torch.Tensor, topk: int, batch: int,
                                     sel_out: torch.Tensor, n_sel_out: torch.Tensor, scores_out: torch.Tensor,
                                     counters: torch.Tensor, *, extra_tokens: int = 1) -> None:
        """fc_score_select of the heads flagged in ``due_mask`` ([L, H] uint8)
        of EVERY layer in one launch, into ``sel_out`` / ``n_sel_out``.
        q_bl: [B, L, Hq, d] (row-major over layers); scores_out:
        [B*L*H, N_cap]; counters: [B*L*H]."""
        _lib.check(self.lib.fc_score_select(
            self._all_layers_view(sel_out, n_sel_out), 0, q_bl.data_ptr(), due_mask.data_ptr(), 1 << 30, 0,
            topk, extra_tokens, 0, scores_out.data_ptr(), counters.data_ptr(), batch, self.stream()),
            "fc_score_select")

    def score_select_into(self, layer: int, q: torch.Tensor, due_mask: torch.Tensor, topk: int, batch: int,
                          sel_out: torch.Tensor, n_sel_out: torch.Tensor, scores_out: torch.Tensor,
                          counters: torch.Tensor, *, extra_tokens: int = 1) -> None:
        """fc_score_select of the heads flagged in ``due_mask`` ([L, H] uint8)
        into the selection buffers ``sel_out`` / ``n_sel_out`` instead of the
        store's own (reload prediction); own scores / counters workspaces."""
        _lib.check(self.lib.fc_score_select(
            self._view_with_sel(sel_out, n_sel_out), layer, q.data_ptr(), due_mask.data_ptr(), 1 << 30, 0,
            topk, extra_tokens, 0, scores_out.data_ptr(), counters.data_ptr(), batch, self.stream()),
            "fc_score_select")

    def fetch_pages_staged(self, layer: int, host_pages: torch.Tensor, copies: torch.Tensor,
                           n_copies: torch.Tensor, staged_map: torch.Tensor, staging: torch.Tensor,
                           n_staged_hits: torch.Tensor | None = None) -> None:
        _lib.check(self.lib.fc_fetch_pages_staged(
            self.cptr, layer, host_pages.data_ptr(), copies.data_ptr(), n_copies.data_ptr(), copies.shape[0],
            staged_map.data_ptr(), staging.data_ptr(), _ptr(n_staged_hits), self.stream()),
            "fc_fetch_pages_staged")

    def stage_promoted(self, pred_sel: torch.Tensor, pred_n: torch.Tensor, unstable: torch.Tensor,
                       slow_resident: torch.Tensor, host_pages: torch.Tensor, staged_map: torch.Tensor,
                       stage_list: torch.Tensor, stage_count: torch.Tensor, staging: torch.Tensor,
                       batch: int) -> None:
        _lib.check(self.lib.fc_stage_promoted(
            self.cptr, pred_sel.data_ptr(), pred_n.data_ptr(), unstable.data_ptr(), slow_resident.data_ptr(),
            host_pages.data_ptr(), staged_map.data_ptr(), stage_list.data_ptr(), stage_count.data_ptr(),
            staging.shape[0], staging.data_ptr(), batch, self.stream()), "fc_stage_promoted")

    def stage_plan(self, pred_sel: torch.Tensor, pred_n: torch.Tensor, unstable: torch.Tensor,
                   slow_resident: torch.Tensor, staged_map: torch.Tensor, stage_list: torch.Tensor,
                   stage_count: torch.Tensor, capacity: int, batch: int, pass_: int = 0) -> None:
        _lib.check(self.lib.fc_stage_plan(
            self.cptr, pred_sel.data_ptr(), pred_n.data_ptr(), unstable.data_ptr(), slow_resident.data_ptr(),
            staged_map.data_ptr(), stage_list.data_ptr(), stage_count.data_ptr(), capacity, batch, pass_,
            self.stream()), "fc_stage_plan")

    def stage_fetch(self, host_pages: torch.Tensor, stage_list: torch.Tensor, stage_count: torch.Tensor,
                    staging: torch.Tensor, pass_: int = 0) -> None:
        _lib.check(self.lib.fc_stage_fetch(self.cptr, host_pages.data_ptr(), stage_list.data_ptr(),
                                           stage_count.data_ptr(), staging.shape[0], staging.data_ptr(), pass_,
                                           self.stream()), "fc_stage_fetch")

    def stage_clear(self, staged_map: torch.Tensor, stage_list: torch.Tensor, stage_count: torch.Tensor,
                    capacity: int) -> None:
        _lib.check(self.lib.fc_stage_clear(self.cptr, staged_map.data_ptr(), stage_list.data_ptr(),
                                           stage_count.data_ptr(), capacity, self.stream()), "fc_stage_clear")

    def fetch_pages(self, layer: int, host_pages: torch.Tensor, copies: torch.Tensor,
                    n_copies: torch.Tensor) -> None:
        _lib.check(self.lib.fc_fetch_pages(self.cptr, layer, host_pages.data_ptr(), copies.data_ptr(),
                                           n_copies.data_ptr(), copies.shape[0], self.stream()),
                   "fc_fetch_pages")

    def offload_filled(self, host_pages: torch.Tensor, unstable: torch.Tensor,
                       slow_resident: torch.Tensor | None, batch: int) -> None:
        _lib.check(self.lib.fc_offload_filled(self.cptr, host_pages.data_ptr(), unstable.data_ptr(),
                                              _ptr(slow_resident), batch, self.stream()),
                   "fc_offload_filled")

    def evict_unselected_row(self, row: int, unstable: torch.Tensor) -> None:
        """fc_evict_unselected of one request row (through its row view)."""
        _lib.check(self.lib.fc_evict_unselected(self.row_view(row), unstable.data_ptr(), 1, self.stream()),
                   "fc_evict_unselected")

    def evict_unselected(self, unstable: torch.Tensor, batch: int) -> None:
        _lib.check(self.lib.fc_evict_unselected(self.cptr, unstable.data_ptr(), batch, self.stream()),
                   "fc_evict_unselected")

    def offload_pages(self, host_pages: torch.Tensor, pages: torch.Tensor, max_ctas: int = 0) -> None:
        _lib.check(self.lib.fc_offload_pages_ctas(self.cptr, host_pages.data_ptr(), pages.data_ptr(),
                                                  pages.shape[0], max_ctas, self.stream()), "fc_offload_pages_ctas")
