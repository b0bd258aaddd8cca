"""Split-context work planner for the persistent decode kernels.

A work unit is a contiguous range of one group's pointer list (group =
(seq, layer, kv_head)).  Units are sized by algorithmic bytes (page header +
code streams + fp16 values, the reference meter formula store.py:315-322),
capped at 1024 tiles, then bin-packed longest-first onto the persistent CTAs;
the unit list is emitted interleaved so the kernel's static `u % grid`
assignment reproduces the bins.  Each group's units own consecutive partial
slots; `slot_begin` drives the LSE merge (the reference's single softmax over
concatenated logits, decode.py:347-354, split flash-decoding style).
"""

from __future__ import annotations

import heapq

import numpy as np

from . import _lib

SM_COUNT = 148
MAX_UNIT_TILES = 512
TILE_ITEMS = 128
PAGE_HEADER_BYTES = 16


class DecodePlan:
    def __init__(self, units, slot_begin, n_slots, grid, group_items, group_ids, dbg_offsets):
        import torch

        self.units_host = units
        self.units = torch.as_tensor(units.view(np.int32).reshape(-1), device="cuda")
        self.n_units = len(units)
        self.slot_begin_host = slot_begin
        self.slot_begin = torch.as_tensor(slot_begin.astype(np.int32), device="cuda")
        self.n_slots = n_slots
        self.grid = grid
        self.group_items = group_items      # retained items per planned group
        self.group_ids = group_ids          # planned groups, merge order
        self.dbg_offsets_host = dbg_offsets
        self.dbg_offsets = torch.as_tensor(dbg_offsets, device="cuda")


def _page_bytes(rows, tiers, d, d_v, P):
    """Algorithmic stream bytes and tiles per page."""
    ab = rows["abits"].astype(np.int64)
    rb = rows["rbits"].astype(np.int64)
    c = rows["count"].astype(np.int64)
    code = (c * (d - 1) * ab + 7) // 8 + (c * rb + 7) // 8
    ti = min(P, TILE_ITEMS)
    return PAGE_HEADER_BYTES + code + 2 * c * d_v, -(-c // ti)


def plan_store(store, groups=None, grid=SM_COUNT, units_per_cta=2) -> DecodePlan:
    """Plan a decode pass over `groups` (default: every group of the store)."""
    n, rows, plen, ptr = store._host()
    if groups is None:
        groups = np.arange(store.groups)
    groups = np.asarray(groups, dtype=np.int64)
    pbytes, ptiles = _page_bytes(rows, store.tiers, store.d, store.d_v, store.page_size)
    lists = [ptr[g, : plen[g]] for g in groups]
    total = sum(int(pbytes[l].sum()) for l in lists)
    target = max(total // max(grid * units_per_cta, 1), 1)
    pieces = []  # (bytes, group, begin, end, piece index)
    for gi, (g, lst) in enumerate(zip(groups, lists)):
        b = pbytes[lst] if len(lst) else np.zeros(0, np.int64)
        t = ptiles[lst] if len(lst) else np.zeros(0, np.int64)
        start, acc, tacc = 0, 0, 0
        for k in range(len(lst)):
            if k > start and (acc + b[k] > target * 1.05 or tacc + t[k] > MAX_UNIT_TILES):
                pieces.append([acc, int(g), start, k])
                start, acc, tacc = k, 0, 0
            acc += int(b[k])
            tacc += int(t[k])
        pieces.append([acc, int(g), start, len(lst)])  # (possibly empty group)
    return _finish(pieces, groups, grid, lambda g: int(rows["count"][ptr[g, : plen[g]]].sum())
                   if plen[g] else 0, lambda g, s, e: int(rows["count"][ptr[g, s:e]].sum())
                   if e > s else 0)


def plan_dense(dstore, groups=None, grid=SM_COUNT, units_per_cta=2) -> DecodePlan:
    """Same planner for the dense baseline store (uniform pages)."""
    G = dstore.batch * dstore.layers * dstore.heads
    if groups is None:
        groups = np.arange(G)
    groups = np.asarray(groups, dtype=np.int64)
    npg = dstore.n_pages_per_group
    P = dstore.page_size
    per_page = PAGE_HEADER_BYTES + P * (dstore.d + dstore.d_v) * 2
    total = len(groups) * npg * per_page
    target = max(total // max(grid * units_per_cta, 1), 1)
    pages_per_unit = max(1, min(int(round(target / per_page)), MAX_UNIT_TILES * 64 // P))
    pieces = []
    for g in groups:
        for s in range(0, max(npg, 1), pages_per_unit):
            e = min(npg, s + pages_per_unit)
            items = min(e * P, dstore.tokens) - s * P
            pieces.append([max(items, 0) * (dstore.d + dstore.d_v) * 2, int(g), s, e])
    T = dstore.tokens
    return _finish(pieces, groups, grid, lambda g: T,
                   lambda g, s, e: max(min(e * P, T) - s * P, 0))


def _finish(pieces, groups, grid, group_items_fn, piece_items_fn):
    # consecutive partial slots per group in `groups` order
    order = {int(g): i for i, g in enumerate(groups)}
    pieces.sort(key=lambda p: (order[p[1]], p[2]))
    slot_begin = np.zeros(len(groups) + 1, dtype=np.int64)
    for i, p in enumerate(pieces):
        p.append(i)  # out_slot
        slot_begin[order[p[1]] + 1] += 1
    slot_begin = np.cumsum(slot_begin)
    n_slots = len(pieces)
    # debug logit offsets (items before this piece in planned-group order)
    gi_items = np.array([group_items_fn(int(g)) for g in groups], dtype=np.int64)
    g_off = np.concatenate([[0], np.cumsum(gi_items)])
    # LPT bin packing onto the CTAs
    grid = max(1, min(grid, len(pieces)))
    heap = [(0, c) for c in range(grid)]
    bins = [[] for _ in range(grid)]
    for p in sorted(pieces, key=lambda p: -p[0]):
        load, c = heapq.heappop(heap)
        bins[c].append(p)
        heapq.heappush(heap, (load + p[0] + 4096, c))
    rounds = max(len(b) for b in bins)
    units, dbg = [], []
    scratch = n_slots  # padding units write here; excluded from the merge
    for r in range(rounds):
        for c in range(grid):
            if r < len(bins[c]):
                _, g, s, e, slot = bins[c][r]
                units.append((g, s, e, slot))
                dbg.append(g_off[order[g]] + piece_items_fn(g, 0, s))
            else:
                units.append((int(groups[0]) if len(groups) else 0, 0, 0, scratch))
                dbg.append(0)
    arr = np.array(units, dtype=np.int32).reshape(-1, 4)
    u = np.zeros(len(arr), dtype=_lib.UNIT_DTYPE)
    u["group"], u["ptr_begin"], u["ptr_end"], u["out_slot"] = arr.T
    return DecodePlan(u, slot_begin, n_slots, grid, gi_items, groups,
                      np.asarray(dbg, dtype=np.int64))
