"""Query-aware page scoring and top-K selection — the reference's
``tierkv.scoring`` API (scoring.py:19-209) backed by the sm_100a kernels.

Per-head objects (``MinMaxMeta``) hold their summaries in a device
``KVStore``; every numeric call runs on the GPU through the C ABI:

* ``update_minmax`` / ``build_minmax``  -> fc_kv_append / fc_kv_prefill
* ``score_pages`` / ``score_page``     -> fc_score_pages
* ``select_topk``                      -> fc_select_topk

Results come back as numpy float64 / tuples, as in the reference.  Scores
are computed in fp32 (the reference uses float64); selection orders fp32
keys exactly like ``np.lexsort((arange, -scores))``.

GQA: ``score_pages`` also accepts a (G, d) query group and returns the
group score sum_g score_pages(q_g).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import HeadId
from .store import PAGE_SIZE, KVStore

META_BLOCK_PAGES = 128  # scoring.py:19


def _device():
    return torch.device("cuda", torch.cuda.current_device())


class MinMaxMeta:
    """Per-page key min/max vectors and fill counts for one head, on the GPU.

    Same public surface as the reference (scoring.py:22-56): ``n_pages``,
    ``add_page``, ``mins``/``maxs`` (float64 host copies; empty pages read
    +inf/-inf), ``fill``, ``blocks_allocated`` (128-page growth).
    """

    def __init__(self, head_dim: int, page_size_tokens: int, *, dtype=torch.float32,
                 _store: KVStore | None = None, _where=(0, 0, 0)):
        if head_dim < 1 or page_size_tokens < 1:
            raise ValueError("head_dim and page_size_tokens must be positive")
        if page_size_tokens != PAGE_SIZE:
            raise ValueError(f"page_size_tokens must be {PAGE_SIZE} on this build")
        self.head_dim = head_dim
        self.page_size_tokens = page_size_tokens
        self.dtype = dtype
        self._store = _store
        self._where = _where  # (row, layer, head) inside the store
        self._n_pages = 0
        self.fill = np.zeros(0, dtype=np.int32)
        self.blocks_allocated = 0

    @classmethod
    def _view(cls, store: KVStore, where, n_tokens: int) -> "MinMaxMeta":
        """Read-only view on the summaries of head ``where`` = (row, layer,
        head) of an existing store holding ``n_tokens`` tokens."""
        meta = cls(store.D, PAGE_SIZE, dtype=store.dtype, _store=store, _where=where)
        n = -(-n_tokens // PAGE_SIZE)
        meta._n_pages = n
        meta.fill = np.full(n, PAGE_SIZE, dtype=np.int32)
        if n:
            meta.fill[-1] = n_tokens - (n - 1) * PAGE_SIZE
        meta.blocks_allocated = -(-n // META_BLOCK_PAGES)
        return meta

    # -- storage -----------------------------------------------------------------

    def _ensure_capacity(self, pages: int) -> None:
        cap = self._store.NCAP if self._store is not None else 0
        if pages <= cap:
            return
        new_cap = -(-pages // META_BLOCK_PAGES) * META_BLOCK_PAGES
        new = KVStore(batch_cap=1, layers=1, kv_heads=1, group=1, head_dim=self.head_dim,
                      pages_cap=new_cap, n_blocks=new_cap + 1, sel_cap=new_cap,
                      dtype=self.dtype, device=_device())
        if self._store is not None:
            old = self._store
            n = self._n_pages
            new.summaries[0, 0, 0, :n] = old.summaries[0, 0, 0, :n]
            # re-home the blocks: logical page p -> block p+1 in the new pool
            blocks = old.table[0, 0, 0, :n].long()
            new.kv_pool[1:n + 1] = old.kv_pool[blocks]
            new.table[0, 0, 0, :n] = torch.arange(1, n + 1, dtype=torch.int32, device=new.device)
            new.free_stack[:new_cap - n] = torch.arange(new_cap, n, -1, dtype=torch.int32,
                                                        device=new.device)
            new.free_top.fill_(new_cap - n)
        self._store = new
        self.blocks_allocated = new_cap // META_BLOCK_PAGES

    @property
    def n_pages(self) -> int:
        return self._n_pages

    def add_page(self) -> int:
        self._ensure_capacity(self._n_pages + 1)
        page = self._n_pages
        self._store.alloc_pages(0, page, 1)
        self.fill = np.append(self.fill, np.int32(0))
        self._n_pages += 1
        return page

    def _check_page(self, page: int) -> None:
        if not 0 <= page < self._n_pages:
            raise ValueError(f"unknown page {page} (have {self._n_pages})")

    def _rows(self, which: int) -> torch.Tensor:
        r, l, h = self._where
        return self._store.summaries[r, l, h, :self._n_pages, which]

    @property
    def mins(self) -> np.ndarray:
        out = self._rows(0).double().cpu().numpy() if self._n_pages else np.empty((0, self.head_dim))
        out[self.fill[:self._n_pages] == 0] = np.inf
        return out

    @property
    def maxs(self) -> np.ndarray:
        out = self._rows(1).double().cpu().numpy() if self._n_pages else np.empty((0, self.head_dim))
        out[self.fill[:self._n_pages] == 0] = -np.inf
        return out


def update_minmax(meta: MinMaxMeta, page: int, key) -> None:
    """Fold one appended key into a page's bounds (scoring.py:59-69) via the
    fused append kernel (fc_kv_append), which writes the key into the page's
    KV block and updates the page summary."""
    meta._check_page(page)
    if meta.fill[page] >= meta.page_size_tokens:
        raise ValueError(f"page {page} is full ({meta.page_size_tokens} keys)")
    key_t = torch.as_tensor(np.asarray(key, dtype=np.float64))
    if tuple(key_t.shape) != (meta.head_dim,):
        raise ValueError(f"key must have shape ({meta.head_dim},)")
    st = meta._store
    dev = st.device
    st.seq_len[0] = page * meta.page_size_tokens + int(meta.fill[page])
    k = key_t.to(dev, st.dtype).reshape(1, 1, -1).contiguous()
    st.append(0, k, torch.zeros_like(k), 1)
    meta.fill[page] += 1


def build_minmax(keys, page_size_tokens: int, *, dtype=torch.float32) -> MinMaxMeta:
    """Vectorised construction from an (n_tokens, d) key matrix
    (scoring.py:72-90) via the prefill kernel (fc_kv_prefill)."""
    keys_t = torch.as_tensor(np.asarray(keys, dtype=np.float64))
    if keys_t.dim() != 2:
        raise ValueError("keys must be (n_tokens, head_dim)")
    n, d = keys_t.shape
    meta = MinMaxMeta(d, page_size_tokens, dtype=dtype)
    if n == 0:
        return meta
    n_pages = -(-n // page_size_tokens)
    meta._ensure_capacity(n_pages)
    meta._store.alloc_pages(0, 0, n_pages)
    k = keys_t.to(meta._store.device, dtype).unsqueeze(0).contiguous()
    meta._store.prefill(0, 0, k, torch.zeros_like(k))
    meta._n_pages = n_pages
    fill = np.full(n_pages, page_size_tokens, dtype=np.int32)
    fill[-1] = n - (n_pages - 1) * page_size_tokens
    meta.fill = fill
    return meta


def _scores_device(q, meta: MinMaxMeta) -> torch.Tensor:
    """fp32 group scores of every page of ``meta`` (device tensor)."""
    st = meta._store
    qn = np.asarray(q, dtype=np.float64)
    qs = qn.reshape(-1, meta.head_dim) if qn.ndim == 2 else qn.reshape(1, meta.head_dim)
    G = qs.shape[0]
    r, l, h = meta._where
    # a temporary descriptor: same buffers, group = G, batch rows up to r
    c = _lib.FcStore.from_buffer_copy(st._c)
    c.group = G
    qt = torch.zeros((r + 1, st.H * G, st.D), dtype=st.dtype, device=st.device)
    qt[r, h * G:(h + 1) * G] = torch.as_tensor(qs).to(st.device, st.dtype)
    saved = st.seq_len[r].clone()
    st.seq_len[r] = meta._n_pages * meta.page_size_tokens  # every page counts as filled
    _lib.check(st.lib.fc_score_pages(ctypes.addressof(c), l, qt.data_ptr(), 0,
                                     st.scores.data_ptr(), r + 1, st.stream()), "fc_score_pages")
    st.seq_len[r] = saved
    return st.scores[r * st.H + h, :meta._n_pages]


def score_pages(q, meta: MinMaxMeta) -> np.ndarray:
    """Scores for every page of one head; all pages must be non-empty
    (scoring.py:102-111)."""
    if meta.n_pages == 0:
        return np.empty(0)
    if (meta.fill[:meta.n_pages] == 0).any():
        raise ValueError("cannot score a head with empty pages")
    return _scores_device(q, meta).double().cpu().numpy()


def score_page(q, meta: MinMaxMeta, page: int) -> float:
    """Upper bound on q·k over the page's keys (scoring.py:93-99)."""
    meta._check_page(page)
    if meta.fill[page] == 0:
        raise ValueError(f"page {page} is empty; nothing to score")
    return float(score_pages(q, meta)[page])


class MinMaxCache:
    """Fast-tier metadata store keyed by (request, layer, head) (scoring.py:114-139)."""

    def __init__(self, head_dim: int, page_size_tokens: int):
        self.head_dim = head_dim
        self.page_size_tokens = page_size_tokens
        self._metas: dict[tuple, MinMaxMeta] = {}

    def get_or_create(self, request_id, head: HeadId) -> MinMaxMeta:
        key = (request_id, HeadId(*head))
        meta = self._metas.get(key)
        if meta is None:
            meta = self._metas[key] = MinMaxMeta(self.head_dim, self.page_size_tokens)
        return meta

    def release_request(self, request_id) -> None:
        for key in [k for k in self._metas if k[0] == request_id]:
            del self._metas[key]

    @property
    def blocks_allocated(self) -> int:
        return sum(m.blocks_allocated for m in self._metas.values())

    def resident_bytes(self, bytes_per_element: int) -> int:
        per_page = 2 * self.head_dim * bytes_per_element
        return sum(m.n_pages * per_page for m in self._metas.values())


@dataclass(frozen=True)
class TopKSet:
    """An ordered selection of page indices for one head (scoring.py:142-161)."""

    pages: tuple
    epoch: int = 0

    def __post_init__(self):
        object.__setattr__(self, "pages", tuple(sorted(int(p) for p in self.pages)))
        if len(set(self.pages)) != len(self.pages):
            raise ValueError("TopKSet pages must be distinct")
        if self.pages and self.pages[0] < 0:
            raise ValueError("TopKSet pages must be non-negative")

    def __contains__(self, page) -> bool:
        return int(page) in set(self.pages)

    def __len__(self) -> int:
        return len(self.pages)


def select_topk_device(scores: torch.Tensor, n_valid: torch.Tensor, k: int, pin_last: bool,
                       out: torch.Tensor, n_out: torch.Tensor) -> None:
    """Batched device select: scores [n_heads, stride] fp32, n_valid [n_heads]."""
    lib = _lib.load()
    _lib.check(lib.fc_select_topk(scores.data_ptr(), scores.shape[1], n_valid.data_ptr(),
                                  scores.shape[0], k, int(pin_last), out.data_ptr(),
                                  n_out.data_ptr(), torch.cuda.current_stream().cuda_stream),
               "fc_select_topk")


def select_topk(scores, k: int, pinned=(), epoch: int = 0) -> TopKSet:
    """Pinned pages plus the highest-scoring others, up to min(k, n_pages);
    ties to the higher score then the lower index (scoring.py:164-193).
    Runs the GPU radix select (fc_select_topk) on fp32 keys."""
    s = np.asarray(scores, dtype=np.float64)
    if s.ndim != 1:
        raise ValueError("scores must be one-dimensional")
    if k < 1:
        raise ValueError("k must be >= 1")
    n = s.size
    pins = sorted({int(p) for p in pinned})
    if pins and (pins[0] < 0 or pins[-1] >= n):
        raise ValueError("pinned pages must reference scored pages")
    if len(pins) > k:
        raise ValueError(f"cannot pin {len(pins)} pages with k={k}")
    if n == 0:
        return TopKSet(pages=(), epoch=epoch)
    dev = _device()
    # the reference's float64 scores as they are (fc_select_topk_f64: exact
    # ranks, no fp32 rounding — distinct float64 scores never become ties)
    st = torch.as_tensor(s, dtype=torch.float64).to(dev)
    pin_last = pins == [n - 1]
    if pins and not pin_last:
        # pinned pages never compete and always enter: give them the top score
        st[torch.as_tensor(pins, device=dev)] = float("inf")
    out = torch.empty(max(k, 1), dtype=torch.int32, device=dev)
    n_out = torch.empty(1, dtype=torch.int32, device=dev)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    lib = _lib.load()
    _lib.check(lib.fc_select_topk_f64(st.data_ptr(), n, k, int(pin_last), ws.data_ptr(), out.data_ptr(),
                                      n_out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
               "fc_select_topk_f64")
    cnt = int(n_out.item())
    return TopKSet(pages=tuple(out[:cnt].tolist()), epoch=epoch)


def rerank_due(head: HeadId, step: int, profile, period: int) -> bool:
    """Unstable heads re-rank every step; stable heads every ``period``
    steps (scoring.py:196-202).  The same rule runs on the device inside
    fc_score_select / fc_rerank_recycle."""
    if period < 1:
        raise ValueError("period must be >= 1")
    if profile.is_unstable(head):
        return True
    return step % period == 0


def layer_scoring_skippable(layer: int, step: int, profile, period: int) -> bool:
    """True when no head in the layer is due (scoring.py:205-209); the decode
    engine uses it to drop the layer's scoring launch from the step."""
    heads = [HeadId(layer, h) for h in range(profile.n_heads_per_layer)]
    return not any(rerank_due(h, step, profile, period) for h in heads)
