"""Serving loop on the real decode path.

The reference's ``Simulator`` (simulator.py:230-600) schedules requests over
a cost model: admission while the committed fast-tier bytes fit
(``_commit_bytes`` / ``_admissible``, simulator.py:253-284), prefill, batched
decode steps, finish, and the ``Metrics`` of simulator.py:87-131.  This loop
keeps that control flow but runs every step on the GPU: requests occupy the
rows of a ``DecodeEngine`` (``start_serving`` / ``admit`` / ``retire``), the
clock advances by the MEASURED device time of each prefill and decode step
(CUDA events), and TTFT / TPOT / throughput come from those times.

With a two-tier engine, admission uses FlexiCache's commit (unstable heads
every page, stable heads their selection, simulator.py:253-266), an
admitted request's full stable-head pages are offloaded after its prefill
on a side stream while decode continues, evicted (and the peak commit
released) once that copy finished and the initial selection exists — reranks
leave the row alone until then — and reranks fetch promoted pages (staged
ahead, tiering.ReloadStager).  With an all-resident engine the
commit is the request's whole KV (simulator.py:257-258).

Each request steps on its own t (simulator.py:437-439): it enters decode at
t = 1 whatever the engine's step, so requests admitted at different times
rerank on different steps (the engine's 'partial' step graphs score only the
rows at their boundary).  With a two-tier engine the reload pause of
simulator.py:321-323,542 is real: a row's promoted pages are fetched on a
side stream after its rerank step and the row is held (emits nothing) until
they landed, while the other rows keep decoding (``reload_pause``; the
metrics report the held fraction of row-steps).  Prompts and
decode inputs are synthetic (the reference has no model either).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, fields

import torch

from .store import PAGE_SIZE


@dataclass
class Request:
    """One request: arrival time (s), prompt and output lengths (tokens)."""
    id: int
    arrival_s: float
    prompt_tokens: int
    output_tokens: int


@dataclass
class ServingMetrics:
    """The reference's ``Metrics`` fields this loop measures (simulator.py:87-131)."""
    n_requests: int = 0
    finished: int = 0
    queued_at_end: int = 0
    total_tokens: int = 0
    output_tokens: int = 0
    sim_time_s: float = 0.0
    throughput_tokens_per_s: float = 0.0
    ttft_mean_s: float = 0.0
    ttft_p50_s: float = 0.0
    ttft_p95_s: float = 0.0
    ttft_p99_s: float = 0.0
    tpot_mean_s: float = 0.0
    tpot_p50_s: float = 0.0
    tpot_p95_s: float = 0.0
    tpot_p99_s: float = 0.0
    peak_batch: int = 0
    peak_fast_bytes: int = 0
    decode_steps: int = 0
    reload_bytes: int = 0
    promoted_fraction: float = 0.0
    pause_steps: int = 0          # row-steps held for a reload (Metrics.pause_steps)
    pause_fraction: float = 0.0   # pause_steps / row-steps of active requests

    def to_text(self) -> str:
        return "".join(f"{f.name} = {getattr(self, f.name)}\n" for f in fields(self))


def _pct(xs, p):
    if not xs:
        return 0.0
    s = sorted(xs)
    k = min(len(s) - 1, max(0, math.ceil(p / 100.0 * len(s)) - 1))
    return s[k]


@dataclass
class _Active:
    req: Request
    row: int
    commit: int = 0
    emitted: int = 0
    first_token_s: float = 0.0
    last_token_s: float = 0.0


class ServingLoop:
    """Continuous batching of ``requests`` over ``engine``'s rows.

    ``make_prompt(req)`` returns (keys, values) [L, H, T, d] on the device;
    ``feed(engine)`` writes the step's q / k_new / v_new (synthetic inputs).
    """

    def __init__(self, engine, requests, make_prompt, feed, *, fast_capacity_blocks: int | None = None,
                 timer=None, reload_pause: bool = True):
        self.eng = engine
        if getattr(engine, "tiering", False) and hasattr(engine, "reload_pause"):
            engine.reload_pause = reload_pause
        self.timer = timer if timer is not None else self._time  # timer(fn) -> seconds
        self.pending = sorted(requests, key=lambda r: (r.arrival_s, r.id))
        self.make_prompt = make_prompt
        self.feed = feed
        st = engine.store
        self.page_bytes = st.page_bytes
        self.LH = engine.L * engine.H
        self.capacity = (st.n_blocks - 1) if fast_capacity_blocks is None else fast_capacity_blocks
        self.committed = 0
        self.now = 0.0
        self.m = ServingMetrics(n_requests=len(requests))
        self._ttft, self._tpot = [], []
        self._rerank_slots = 0
        self._row_steps = 0
        self._captured = False

    def _commit_blocks(self, req: Request) -> int:
        n_max = (req.prompt_tokens + req.output_tokens) // PAGE_SIZE + 1
        if not self.eng.tiering:
            # all-resident: every page the request will ever hold, for every
            # (layer, head) (DENSE commit, simulator.py:257-258)
            return n_max * self.LH
        # two-tier (FlexiCache commit, simulator.py:253-266): unstable heads keep
        # every page, stable heads their selection + the pages appended between
        # reranks; at least the prompt until its post-prefill eviction
        n_unstable = int(self.eng.unstable.sum().item())
        n_stable = self.LH - n_unstable
        slack = self.eng.R // PAGE_SIZE + 2
        steady = n_unstable * n_max + n_stable * (min(self.eng.K, n_max) + slack)
        peak = (req.prompt_tokens // PAGE_SIZE + 1 + slack) * self.LH
        return max(steady, peak)

    def _steady_blocks(self, req: Request) -> int:
        """The commitment once the prompt's unselected stable-head pages left
        HBM (_finish_prefill_offload releases the rest, simulator.py:389-408)."""
        if not self.eng.tiering:
            return self._commit_blocks(req)
        n_max = (req.prompt_tokens + req.output_tokens) // PAGE_SIZE + 1
        n_unstable = int(self.eng.unstable.sum().item())
        slack = self.eng.R // PAGE_SIZE + 2
        return n_unstable * n_max + (self.LH - n_unstable) * (min(self.eng.K, n_max) + slack)

    def _time(self, fn) -> float:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / 1e3

    def run(self, max_steps: int = 1 << 30) -> ServingMetrics:
        eng = self.eng
        eng.start_serving()
        free_rows = list(range(eng.B))
        active: dict[int, _Active] = {}
        ready: list[Request] = []
        steps = 0
        while (self.pending or ready or active) and steps < max_steps:
            while self.pending and self.pending[0].arrival_s <= self.now:
                ready.append(self.pending.pop(0))
            # admission while a row is free and the commitment fits (_admissible)
            while ready and free_rows:
                need = self._commit_blocks(ready[0])
                if need > self.capacity:
                    raise ValueError(f"request {ready[0].id} cannot fit even alone ({need} blocks)")
                if self.committed + need > self.capacity:
                    break
                req = ready.pop(0)
                row = free_rows.pop(0)
                self.committed += need
                keys, values = self.make_prompt(req)
                self.now += self.timer(lambda: eng.admit(row, keys, values))
                if not self._captured and hasattr(eng, "capture_graphs"):
                    # one-time setup outside the clock (as bench.py captures
                    # before its timed region): the step graphs
                    eng.capture_graphs(("plain", "rerank", "partial"))
                    self._captured = True
                active[row] = _Active(req, row, commit=need)
                self._ttft.append(self.now - req.arrival_s)  # prefill emits the first token
                active[row].emitted = 1
                active[row].first_token_s = active[row].last_token_s = self.now
                self.m.total_tokens += req.prompt_tokens
            self.m.peak_batch = max(self.m.peak_batch, len(active))
            in_use = (eng.store.n_blocks - 1 - eng.store.free_count()) * self.page_bytes
            self.m.peak_fast_bytes = max(self.m.peak_fast_bytes, in_use)
            if not active:  # idle: jump to the next arrival
                if self.pending:
                    self.now = max(self.now, self.pending[0].arrival_s)
                continue
            self.feed(eng)
            pre_seq = list(getattr(eng, "seq_host", ()))
            dt = self.timer(eng.step)
            eng.store.check_errors()
            self.now += dt
            steps += 1
            if eng.tiering:
                # rerank slots of rows that recycled (simulator.py:532): stable
                # heads x their target, rows past their post-prefill offload
                n_stable = self.LH - int(eng.unstable.sum().item())
                reranked = getattr(eng, "rerank_rows", None)
                if reranked is None:
                    reranked = list(active) if eng.is_rerank_step() else []
                for row in reranked:
                    if row in active and not eng.eviction_pending(row):
                        pages = (pre_seq[row] + 1 + PAGE_SIZE - 1) // PAGE_SIZE
                        self._rerank_slots += n_stable * min(eng.K, pages)
            decoded = getattr(eng, "decoded_rows", None)
            decoded = set(active) if decoded is None else set(decoded)
            self._row_steps += len(active)
            self.m.pause_steps += len(set(active) - decoded)
            for row in list(active):
                if row not in decoded:  # held for its reload: no token this step
                    continue
                a = active[row]
                a.emitted += 1
                a.last_token_s = self.now
                self.m.output_tokens += 1
                steady = self._steady_blocks(a.req)
                if a.commit > steady and not eng.eviction_pending(row):
                    # selected, offloaded and evicted: the peak is released
                    self.committed -= a.commit - steady
                    a.commit = steady
                if a.emitted >= a.req.output_tokens:
                    # timed: a two-tier row still offloading waits for that copy here
                    self.now += self.timer(lambda: eng.retire(row))
                    self.committed -= a.commit
                    free_rows.append(row)
                    if a.emitted > 1:
                        # per request, as the reference's _finish (simulator.py:590-592):
                        # (last - first token) / (emitted - 1), so prefills of other
                        # requests and retires between its tokens count
                        self._tpot.append((a.last_token_s - a.first_token_s) / (a.emitted - 1))
                    self.m.finished += 1
                    del active[row]
        m = self.m
        m.queued_at_end = len(self.pending) + len(ready)
        m.decode_steps = steps
        m.pause_fraction = m.pause_steps / self._row_steps if self._row_steps else 0.0
        m.sim_time_s = self.now
        m.throughput_tokens_per_s = m.output_tokens / self.now if self.now > 0 else 0.0
        if eng.tiering:  # promoted pages fetched over the host link (simulator.py:535-541, :600)
            promoted = int(eng.fetched_pages.item())
            m.reload_bytes = promoted * self.page_bytes
            m.promoted_fraction = promoted / self._rerank_slots if self._rerank_slots else 0.0
        if self._ttft:
            m.ttft_mean_s = sum(self._ttft) / len(self._ttft)
            m.ttft_p50_s, m.ttft_p95_s, m.ttft_p99_s = (_pct(self._ttft, p) for p in (50, 95, 99))
        if self._tpot:
            m.tpot_mean_s = sum(self._tpot) / len(self._tpot)
            m.tpot_p50_s, m.tpot_p95_s, m.tpot_p99_s = (_pct(self._tpot, p) for p in (50, 95, 99))
        return m
