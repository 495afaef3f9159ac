"""GPU-resident page table and physical pool — the reference's
``tierkv.blocktable`` API (blocktable.py:28-465) on the device free list.

The table ``[requests_cap, L, H, pages_cap]`` int32 and the LIFO free stack
live in device memory and are mutated only by the library kernels:

* ``allocate_page(s)``          -> fc_alloc_pages on a one-head view
* ``allocate_page_all_heads``   -> fc_alloc_pages ((layer, head) order)
* ``evict_to_null`` / ``evict_many`` / ``release_request`` -> fc_evict_pages
* ``recycle``                   -> fc_rerank_recycle on a one-head view

Host-side validation mirrors the reference (same exceptions, raised before
any mutation); lookups read the table back.  The dirty-run shadow copy
(``flush_dirty``) is not part of the per-step path: the
table is GPU-authoritative.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import HeadId
from .errors import ConsistencyError, PoolExhausted

NULL_BLOCK = 0  # blocktable.py:25


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


class PhysicalPool:
    """Flat block pool with a reserved null block and a LIFO free list on the
    device (blocktable.py:28-94).  A fresh pool pops 1, 2, 3, ..."""

    def __init__(self, total_blocks: int, tier: str = "fast"):
        if total_blocks < 2:
            raise ValueError("pool needs at least one real block beyond the null block")
        if tier not in ("fast", "slow"):
            raise ValueError(f"unknown tier {tier!r}")
        self.tier = tier
        self.total_blocks = total_blocks
        dev = _dev()
        self.free_stack = torch.zeros(total_blocks, dtype=torch.int32, device=dev)
        self.free_stack[:total_blocks - 1] = torch.arange(total_blocks - 1, 0, -1, dtype=torch.int32)
        self.free_top = torch.tensor([total_blocks - 1], dtype=torch.int32, device=dev)

    @property
    def free_count(self) -> int:
        return int(self.free_top.item())

    @property
    def live_count(self) -> int:
        return self.total_blocks - 1 - self.free_count

    def free_list(self) -> list:
        """Free blocks bottom..top (the reference's ``_free`` order)."""
        return self.free_stack[:self.free_count].tolist()

    def clone(self) -> "PhysicalPool":
        new = PhysicalPool.__new__(PhysicalPool)
        new.tier, new.total_blocks = self.tier, self.total_blocks
        new.free_stack, new.free_top = self.free_stack.clone(), self.free_top.clone()
        return new


@dataclass(frozen=True)
class RecyclePlan:
    """Outcome of one re-rank's block shuffle for a single head (blocktable.py:97-106)."""

    evicted: tuple
    promoted: tuple
    reassigned: tuple
    freed_blocks: tuple
    fresh_allocs: tuple
    copies: tuple


class BlockTable:
    """Dense (request, layer, head, logical page) -> physical block mapping
    (blocktable.py:109-440), GPU-resident."""

    def __init__(self, pool: PhysicalPool, num_layers: int, kv_heads_per_layer: int, *,
                 requests_cap: int = 4, pages_cap: int = 8):
        if num_layers < 1 or kv_heads_per_layer < 1:
            raise ValueError("layer and head counts must be positive")
        self.pool = pool
        self.L, self.H = num_layers, kv_heads_per_layer
        dev = _dev()
        self._table = torch.zeros((requests_cap, self.L, self.H, pages_cap), dtype=torch.int32, device=dev)
        self._n_pages = np.zeros((requests_cap, self.L, self.H), dtype=np.int32)
        self._rows: dict = {}
        self._free_rows = list(range(requests_cap - 1, -1, -1))
        # scratch for one-head views (selection rows, counts, seq_len, copy list, error word)
        self._scratch = torch.zeros(64, dtype=torch.int32, device=dev)
        self._err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._step = torch.zeros(1, dtype=torch.int32, device=dev)
        self._dummy = torch.zeros(256, dtype=torch.float32, device=dev)
        self._unstable0 = torch.zeros(1, dtype=torch.uint8, device=dev)
        self.lib = _lib.load()

    # -- shape bookkeeping ---------------------------------------------------------

    @property
    def shape(self):
        return tuple(self._table.shape)

    def _grow_pages(self, need: int) -> None:
        cap = self._table.shape[3]
        new_cap = max(cap * 2, need)
        pad = torch.zeros(self._table.shape[:3] + (new_cap - cap,), dtype=torch.int32,
                          device=self._table.device)
        self._table = torch.cat([self._table, pad], dim=3).contiguous()

    def _grow_rows(self) -> None:
        cap = self._table.shape[0]
        pad = torch.zeros((cap,) + self._table.shape[1:], dtype=torch.int32, device=self._table.device)
        self._table = torch.cat([self._table, pad], dim=0).contiguous()
        self._n_pages = np.concatenate([self._n_pages, np.zeros_like(self._n_pages)])
        self._free_rows = list(range(2 * cap - 1, cap - 1, -1)) + self._free_rows

    def add_request(self, request_id) -> int:
        if request_id in self._rows:
            raise ConsistencyError(f"request {request_id!r} already registered")
        if not self._free_rows:
            self._grow_rows()
        row = self._free_rows.pop()
        self._rows[request_id] = row
        return row

    def _row(self, request_id) -> int:
        try:
            return self._rows[request_id]
        except KeyError:
            raise ConsistencyError(f"unknown request {request_id!r}") from None

    # -- device views ----------------------------------------------------------------

    def _view(self, row: int, layer: int = 0, head: int = 0, *, all_heads: bool = False):
        """fc_store descriptor over this table + pool: the whole table
        (all_heads) or a single (row, layer, head) row as a 1x1x1 store."""
        t = self._table
        N = t.shape[3]
        if all_heads:
            B, L, H, table_ptr = t.shape[0], self.L, self.H, t.data_ptr()
        else:
            B, L, H = 1, 1, 1
            table_ptr = t.data_ptr() + (((row * self.L + layer) * self.H + head) * N) * 4
        sc = self._scratch
        st = _lib.FcStore(B, L, H, 1, 64, 16, N, 32, _lib.FC_F32, self.pool.total_blocks,
                          self._dummy.data_ptr(), self._dummy.data_ptr(), table_ptr,
                          sc.data_ptr() + 0 * 4,           # seq_len
                          sc[8:].data_ptr(),               # sel (unused by table ops)
                          sc[4:].data_ptr(),               # n_sel
                          self.pool.free_stack.data_ptr(), self.pool.free_top.data_ptr(),
                          self._step.data_ptr(), self._err.data_ptr())
        return st

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def _check_device_errors(self):
        bits = int(self._err.item())
        if bits:
            self._err.zero_()
            if bits & _lib.FC_ERR_POOL_EXHAUSTED:
                raise PoolExhausted(f"{self.pool.tier} pool exhausted")
            raise ConsistencyError(f"device error bits {bits:#x}")

    # -- lookups -----------------------------------------------------------------------

    def n_pages(self, request_id, head: HeadId) -> int:
        return int(self._n_pages[self._row(request_id), head[0], head[1]])

    def _row_entries(self, row, l, h) -> np.ndarray:
        n = int(self._n_pages[row, l, h])
        return self._table[row, l, h, :n].cpu().numpy()

    def physical(self, request_id, head: HeadId, logical: int) -> int:
        row = self._row(request_id)
        if not 0 <= logical < self._n_pages[row, head[0], head[1]]:
            raise ValueError(f"logical page {logical} not allocated for {head}")
        return int(self._table[row, head[0], head[1], logical].item())

    def physical_for_read(self, request_id, head: HeadId, logical: int) -> int:
        block = self.physical(request_id, head, logical)
        if block == NULL_BLOCK:
            raise ConsistencyError(f"read of evicted page {logical} for {head}: null block is not data")
        return block

    def resident_pages(self, request_id, head: HeadId) -> np.ndarray:
        row = self._row(request_id)
        return np.flatnonzero(self._row_entries(row, head[0], head[1]) != NULL_BLOCK)

    def assert_resident(self, request_id, head: HeadId, pages) -> None:
        row = self._row(request_id)
        pages = np.asarray(list(pages), dtype=np.int64)
        if pages.size == 0:
            return
        n = self._n_pages[row, head[0], head[1]]
        if pages.min() < 0 or pages.max() >= n:
            raise ValueError("page index out of allocated range")
        entries = self._row_entries(row, head[0], head[1])[pages]
        if (entries == NULL_BLOCK).any():
            raise ConsistencyError(f"pages {pages[entries == NULL_BLOCK].tolist()} of {head} "
                                   "are not fast-tier resident")

    # -- mutation ----------------------------------------------------------------------

    def allocate_pages(self, request_id, head: HeadId, count: int) -> np.ndarray:
        """blocktable.py:236-246 — one head's pages, blocks in pop order."""
        row = self._row(request_id)
        l, h = head[0], head[1]
        n = int(self._n_pages[row, l, h])
        if n + count > self._table.shape[3]:
            self._grow_pages(n + count)
        if count > self.pool.free_count:
            raise PoolExhausted(f"{self.pool.tier} pool exhausted: need {count}, "
                                f"have {self.pool.free_count} free")
        st = self._view(row, l, h)
        _lib.check(self.lib.fc_alloc_pages(ctypes.byref(st), 0, n, count, self._stream()),
                   "fc_alloc_pages")
        self._check_device_errors()
        self._n_pages[row, l, h] = n + count
        return np.arange(n, n + count)

    def allocate_page(self, request_id, head: HeadId) -> int:
        """blocktable.py:223-234."""
        return int(self.allocate_pages(request_id, head, 1)[0])

    def allocate_page_all_heads(self, request_id) -> int:
        """blocktable.py:248-263: the same new logical page for every head,
        blocks handed out in (layer, head) order."""
        row = self._row(request_id)
        counts = self._n_pages[row]
        n = int(counts.reshape(-1)[0])
        if (counts != n).any():
            raise ConsistencyError("heads disagree on page count; cannot append in lockstep")
        if n == self._table.shape[3]:
            self._grow_pages(n + 1)
        if self.L * self.H > self.pool.free_count:
            raise PoolExhausted(f"{self.pool.tier} pool exhausted")
        st = self._view(row, all_heads=True)
        _lib.check(self.lib.fc_alloc_pages(ctypes.byref(st), row, n, 1, self._stream()), "fc_alloc_pages")
        self._check_device_errors()
        self._n_pages[row] = n + 1
        return n

    def _evict_list(self, entries) -> None:
        if not entries:
            return
        t = torch.tensor(entries, dtype=torch.int32, device=self._table.device).reshape(-1, 4)
        st = self._view(0, all_heads=True)
        _lib.check(self.lib.fc_evict_pages(ctypes.byref(st), t.data_ptr(), t.shape[0], self._stream()),
                   "fc_evict_pages")
        self._check_device_errors()

    def evict_to_null(self, request_id, head: HeadId, logical: int) -> int:
        """blocktable.py:265-278."""
        row = self._row(request_id)
        l, h = head[0], head[1]
        if not 0 <= logical < self._n_pages[row, l, h]:
            raise ValueError(f"logical page {logical} not allocated for {head}")
        block = int(self._table[row, l, h, logical].item())
        if block == NULL_BLOCK:
            raise ConsistencyError(f"double eviction of page {logical} for {head}")
        self._evict_list([row, l, h, logical])
        return block

    def evict_many(self, request_id, head: HeadId, logicals) -> np.ndarray:
        """blocktable.py:280-294: releases in ascending page order."""
        row = self._row(request_id)
        l, h = head[0], head[1]
        pages = np.asarray(sorted(int(p) for p in logicals), dtype=np.int64)
        if pages.size == 0:
            return np.empty(0, dtype=np.int32)
        if pages[0] < 0 or pages[-1] >= self._n_pages[row, l, h]:
            raise ValueError("logical page out of allocated range")
        blocks = self._row_entries(row, l, h)[pages]
        if (blocks == NULL_BLOCK).any():
            raise ConsistencyError("double eviction within batch")
        self._evict_list([v for p in pages for v in (row, l, h, int(p))])
        return blocks.astype(np.int32)

    def release_request(self, request_id) -> int:
        """blocktable.py:161-172: free every live block of a request."""
        row = self._row(request_id)
        entries = []
        for l in range(self.L):
            for h in range(self.H):
                live = np.flatnonzero(self._row_entries(row, l, h) != NULL_BLOCK)
                entries += [v for p in live for v in (row, l, h, int(p))]
        self._evict_list(entries)
        self._n_pages[row] = 0
        del self._rows[request_id]
        self._free_rows.append(row)
        return len(entries) // 4

    def recycle(self, request_id, head: HeadId, old_topk, new_topk, slow_resident=None) -> RecyclePlan:
        """blocktable.py:296-357 on the device: evicted = old \\ new and
        promoted = new \\ old paired in ascending order (fc_rerank_recycle)."""
        row = self._row(request_id)
        l, h = head[0], head[1]
        old = np.unique(np.asarray(list(old_topk), dtype=np.int64))
        new = np.unique(np.asarray(list(new_topk), dtype=np.int64))
        n = int(self._n_pages[row, l, h])
        for arr, name in ((old, "old"), (new, "new")):
            if arr.size and (arr[0] < 0 or arr[-1] >= n):
                raise ValueError(f"{name} selection references unallocated pages")
        before = self._row_entries(row, l, h)
        evicted = np.setdiff1d(old, new, assume_unique=True)
        promoted = np.setdiff1d(new, old, assume_unique=True)
        if old.size and (before[old] == NULL_BLOCK).any():
            raise ConsistencyError("old selection references evicted pages")
        if promoted.size and (before[promoted] != NULL_BLOCK).any():
            raise ConsistencyError("promoted page is already resident")
        if slow_resident is not None:
            srs = {int(p) for p in slow_resident}
            missing = [int(p) for p in promoted if int(p) not in srs]
            if missing:
                raise ConsistencyError(f"promoted pages {missing} have no slow-tier copy for {head}")
        m = min(evicted.size, promoted.size)
        if promoted.size - m > self.pool.free_count:
            raise PoolExhausted(f"{self.pool.tier} pool exhausted")
        dev = self._table.device
        cap = max(old.size, new.size, 1)
        old_sel = torch.zeros(cap, dtype=torch.int32, device=dev)
        old_sel[:old.size] = torch.as_tensor(old, dtype=torch.int32)
        n_old = torch.tensor([old.size], dtype=torch.int32, device=dev)
        new_sel = torch.zeros(cap, dtype=torch.int32, device=dev)
        new_sel[:new.size] = torch.as_tensor(new, dtype=torch.int32)
        n_new = torch.tensor([new.size], dtype=torch.int32, device=dev)
        seq = torch.tensor([n * 16], dtype=torch.int32, device=dev)
        copies = torch.zeros((max(promoted.size, 1), 4), dtype=torch.int32, device=dev)
        n_copies = torch.zeros(1, dtype=torch.int32, device=dev)
        st = self._view(row, l, h)
        st.sel_cap = cap
        ws = torch.zeros(self.lib.fc_rerank_workspace_size(ctypes.byref(st)) // 4, dtype=torch.int32, device=dev)
        st.sel, st.n_sel, st.seq_len = new_sel.data_ptr(), n_new.data_ptr(), seq.data_ptr()
        _lib.check(self.lib.fc_rerank_recycle(
            ctypes.byref(st), 0, old_sel.data_ptr(), n_old.data_ptr(), self._unstable0.data_ptr(),
            1, 1, 0, 0, None, copies.data_ptr(), copies.shape[0], n_copies.data_ptr(),
            ws.data_ptr(), 1, self._stream()), "fc_rerank_recycle")
        self._check_device_errors()
        nc = int(n_copies.item())
        cp = copies[:nc].cpu().numpy()
        cp = cp[np.argsort(cp[:, 2], kind="stable")]
        copy_list = tuple((int(p), int(b)) for p, b in zip(cp[:, 2], cp[:, 3]))
        reassigned = tuple((int(e), int(p), int(before[e])) for e, p in zip(evicted[:m], promoted[:m]))
        freed = tuple(int(before[e]) for e in evicted[m:])
        dest = dict(copy_list)
        fresh = tuple((int(p), dest[int(p)]) for p in promoted[m:])
        return RecyclePlan(evicted=tuple(int(p) for p in evicted), promoted=tuple(int(p) for p in promoted),
                           reassigned=reassigned, freed_blocks=freed, fresh_allocs=fresh, copies=copy_list)

    # -- invariants ------------------------------------------------------------------

    def live_entries(self) -> np.ndarray:
        t = self._table.cpu().numpy()
        return t[t != NULL_BLOCK]

    def check_injective(self) -> None:
        live = self.live_entries()
        if np.unique(live).size != live.size:
            raise ConsistencyError("physical block mapped by two logical pages")

    def check_conservation(self) -> None:
        live = self.live_entries().size
        if self.pool.live_count != live:
            raise ConsistencyError(f"pool live count {self.pool.live_count} != table live entries {live}")

    def clone(self) -> "BlockTable":
        new = BlockTable.__new__(BlockTable)
        new.__dict__.update(self.__dict__)
        new.pool = self.pool.clone()
        new._table = self._table.clone()
        new._n_pages = self._n_pages.copy()
        new._rows = dict(self._rows)
        new._free_rows = list(self._free_rows)
        new._scratch = self._scratch.clone()
        new._err = torch.zeros_like(self._err)
        return new

    def canonical_form(self) -> np.ndarray:
        """Table with physical ids relabelled in first-appearance order (blocktable.py:414-428)."""
        flat = self._table.cpu().numpy().reshape(-1)
        out = np.zeros_like(flat)
        mapping = {NULL_BLOCK: NULL_BLOCK}
        for pos in np.flatnonzero(flat):
            b = int(flat[pos])
            if b not in mapping:
                mapping[b] = len(mapping)
            out[pos] = mapping[b]
        return out.reshape(self._table.shape)
