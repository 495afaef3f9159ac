"""Serving-loop control flow (admission under the fast-tier budget, finish,
metrics) with a stand-in engine — no GPU (the loop itself is host code;
tests/test_gpu_serving.py runs it on the decode path)."""

from paper_2511_00868_b200.serving import Request, ServingLoop


class _Store:
    def __init__(self, n_blocks):
        self.n_blocks = n_blocks
        self.used = 0
        self.page_bytes = 8192

    def free_count(self):
        return self.n_blocks - 1 - self.used

    def check_errors(self):
        pass


class _Engine:
    """Rows, prefill / free bookkeeping and a step counter, no kernels."""

    def __init__(self, B, L, H, n_blocks):
        self.B, self.L, self.H = B, L, H
        self.tiering = False
        self.store = _Store(n_blocks)
        self.rows = {}
        self.steps = 0
        self.max_active = 0

    def start_serving(self):
        self.rows = {}

    def admit(self, row, keys, values):
        assert row not in self.rows
        T = keys
        self.rows[row] = T
        self.store.used += (T // 16 + 1) * self.L * self.H

    def retire(self, row):
        T = self.rows.pop(row)
        self.store.used -= (T // 16 + 1) * self.L * self.H

    def step(self):
        self.steps += 1
        self.max_active = max(self.max_active, len(self.rows))


def _run(requests, B=2, n_blocks=10_000, step_s=0.01, prefill_s=0.05):
    eng = _Engine(B, 2, 2, n_blocks)
    times = iter([])

    def timer(fn):
        name = getattr(fn, "__name__", "")
        fn()
        if "retire" in getattr(getattr(fn, "__code__", None), "co_names", ()):
            return 0.0  # freeing a row: no device time in this stand-in
        return step_s if name == "step" else prefill_s
    loop = ServingLoop(eng, requests, make_prompt=lambda r: (r.prompt_tokens, r.prompt_tokens),
                       feed=lambda e: None, timer=timer)
    del times
    return loop.run(), eng


def test_every_request_finishes_and_tokens_add_up():
    reqs = [Request(i, 0.0, 100 + 10 * i, 5 + i) for i in range(5)]
    m, eng = _run(reqs, B=2)
    assert m.finished == 5 and m.queued_at_end == 0
    assert m.output_tokens == sum(r.output_tokens - 1 for r in reqs)  # prefill emits the first token
    assert m.peak_batch == 2 and eng.max_active == 2
    assert eng.rows == {}
    assert m.throughput_tokens_per_s > 0 and m.tpot_mean_s >= 0.01


def test_tpot_is_per_request_and_counts_other_prefills():
    # simulator.py:590-592: TPOT = (last - first token) / (emitted - 1) per
    # request, so another request's prefill between two tokens counts
    reqs = [Request(0, 0.0, 100, 10), Request(1, 0.03, 100, 3)]
    m, _ = _run(reqs, B=2)
    a = (0.05 + 0.05 + 9 * 0.01 - 0.05) / 9      # first token 0.05, B's prefill, 9 steps
    b = 0.01                                      # first token 0.10, 2 steps
    assert abs(m.tpot_mean_s - (a + b) / 2) < 1e-12
    assert abs(m.tpot_p95_s - a) < 1e-12 and abs(m.tpot_p50_s - b) < 1e-12


def test_admission_waits_for_budget():
    # each request commits (160 // 16 + 1) * 4 = 44 blocks: the budget holds one
    reqs = [Request(i, 0.0, 150, 3) for i in range(3)]
    m, eng = _run(reqs, B=3, n_blocks=60)
    assert m.finished == 3 and m.peak_batch == 1


def test_idle_until_arrival_and_ttft():
    reqs = [Request(0, 1.0, 64, 2)]
    m, _ = _run(reqs, B=1)
    assert m.finished == 1
    assert abs(m.ttft_mean_s - 0.05) < 1e-12          # arrives at 1.0, prefilled by 1.05
    assert abs(m.sim_time_s - (1.0 + 0.05 + 0.01)) < 1e-12


class _TieredEngine(_Engine):
    """Two-tier stand-in: a request's post-prefill offload takes `lag` steps;
    its eviction (and the loop's release of the peak commit) waits for it."""

    def __init__(self, B, L, H, n_blocks, lag):
        super().__init__(B, L, H, n_blocks)
        self.tiering = True
        self.K, self.R = 2, 4
        self.lag = lag
        self.pending = {}
        self.seq_host = [-1] * B
        import torch
        self.unstable = torch.zeros(L * H, dtype=torch.uint8)
        self.fetched_pages = torch.zeros(1, dtype=torch.int64)
        self.commit_log = []

    def admit(self, row, keys, values):
        super().admit(row, keys, values)
        self.pending[row] = self.steps + self.lag
        self.seq_host[row] = keys

    def retire(self, row):
        super().retire(row)
        self.pending.pop(row, None)
        self.seq_host[row] = -1

    def eviction_pending(self, row):
        return row in self.pending

    def is_rerank_step(self):
        return (self.steps + 1) % self.R == 0

    def step(self):
        super().step()
        for row, t in list(self.pending.items()):
            if self.steps >= t:
                del self.pending[row]


def test_tiered_peak_commit_held_until_offload_lands():
    """FlexiCache commit: the peak (whole prompt) stays committed while the
    post-prefill offload is in flight and drops to the steady commit after
    (simulator.py:389-408); a second request that only fits at steady state
    is admitted only then."""
    from paper_2511_00868_b200.serving import ServingLoop
    eng = _TieredEngine(2, 2, 2, n_blocks=10_000, lag=3)
    reqs = [Request(0, 0.0, 320, 12), Request(1, 0.0, 320, 4)]
    loop = ServingLoop(eng, reqs, make_prompt=lambda r: (r.prompt_tokens, r.prompt_tokens),
                       feed=lambda e: None, timer=lambda fn: (fn(), 0.01)[1])
    peak, steady = loop._commit_blocks(reqs[0]), loop._steady_blocks(reqs[0])
    assert peak > steady
    loop.capacity = peak + steady  # both fit only once the first is at its steady commit
    admitted_at = {}
    orig_admit = eng.admit

    def admit(row, keys, values):
        admitted_at[row] = eng.steps
        orig_admit(row, keys, values)
    eng.admit = admit
    m = loop.run()
    assert m.finished == 2
    assert admitted_at[0] == 0 and admitted_at[1] >= eng.lag  # waited for request 0's offload
    assert loop.committed == 0


class _PausingEngine(_Engine):
    """Stand-in whose rows are held one step at each of their own 4th steps
    (the reload pause): a held row emits nothing that step."""

    def __init__(self, *a):
        super().__init__(*a)
        self.t_row = {}
        self.decoded_rows = []

    def admit(self, row, keys, values):
        super().admit(row, keys, values)
        self.t_row[row] = 1

    def retire(self, row):
        super().retire(row)
        self.t_row.pop(row, None)

    def step(self):
        super().step()
        self.decoded_rows = []
        for row, t in self.t_row.items():
            if t % 4 == 0 and not getattr(self, "_held", {}).get(row):
                self.__dict__.setdefault("_held", {})[row] = True  # held once at its boundary
                continue
            self.__dict__.setdefault("_held", {})[row] = False
            self.decoded_rows.append(row)
            self.t_row[row] = t + 1


def test_held_rows_emit_nothing_and_the_pause_fraction_counts_them():
    """simulator.py:321-323,542: a reloading request does not step; the
    others do.  Tokens add up, and Metrics.pause_steps counts the held
    row-steps."""
    eng = _PausingEngine(2, 2, 2, 10_000)
    reqs = [Request(0, 0.0, 100, 9), Request(1, 0.0, 120, 9)]
    loop = ServingLoop(eng, reqs, make_prompt=lambda r: (r.prompt_tokens, r.prompt_tokens),
                       feed=lambda e: None, timer=lambda fn: (fn(), 0.01)[1])
    m = loop.run()
    assert m.finished == 2
    assert m.output_tokens == 2 * 8
    # 8 decoded tokens per request with a hold at t = 4 and t = 8 -> 10 steps each
    assert m.pause_steps == 4 and m.decode_steps == 10
    assert abs(m.pause_fraction - 4 / 20) < 1e-12
