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

import os

import numpy as np

from . import _lib

SM_COUNT = 148
MAX_UNIT_TILES = 512   # defaults; the built library's values win (tile_geometry)
TILE_ITEMS = 128
_GEOM = None


def tile_geometry():
    """(items per ADA tile, tile cap per unit) of the loaded library
    (sphkv_ada_tile_items / sphkv_unit_tile_cap)."""
    global _GEOM
    if _GEOM is None:
        l = _lib.lib()
        _GEOM = (int(l.sphkv_ada_tile_items()), int(l.sphkv_unit_tile_cap()))
    return _GEOM
PAGE_HEADER_BYTES = 16


class DecodePlan:
    def __init__(self, units, slot_begin, n_slots, grid, group_items, group_ids, dbg_offsets,
                 slot_group=None, dynamic=False):
        import torch

        self.units_host = units
        # plan metadata lives on the device the kernels run on; on a host
        # without CUDA (planner unit tests) it stays in host memory -- every
        # decode entry point still requires the GPU (_lib.require_gpu)
        dev = "cuda" if torch.cuda.is_available() else "cpu"
        self.units = torch.as_tensor(units.view(np.int32).reshape(-1), device=dev)
        self.n_units = len(units)
        self.slot_begin_host = slot_begin
        self.slot_begin = torch.as_tensor(slot_begin.astype(np.int32), device=dev)
        self.n_slots = n_slots
        self.grid = grid
        self.group_items = group_items      # retained items per planned group
        self.group_ids = group_ids          # planned groups, merge order
        self.dbg_offsets_host = dbg_offsets
        self.dbg_offsets = torch.as_tensor(dbg_offsets, device=dev)
        self.dynamic = dynamic
        # fused in-kernel merge: plan group of every partial slot (+ scratch = -1)
        # and the caller-zeroed control words (sphkv_ada_decode_fused)
        sg = np.full(n_slots + 1, -1, dtype=np.int32)
        if slot_group is not None:
            sg[:n_slots] = slot_group
        self.slot_group = torch.as_tensor(sg, device=dev)
        # [groups] split counters, queue head, CTAs done, error word (a unit
        # over the kernel's tile list: SPHKV_E_CAPACITY)
        self.ctl = torch.zeros(len(group_ids) + 3, dtype=torch.int32, device=dev)
        # planner-made units respect the tile cap; set for hand-made plans
        self.check_units = False


def _page_bytes(rows, tiers, d, d_v, P):
    """Algorithmic stream bytes and tiles per page."""
    ab = rows["abits"].astype(np.int64)
    rb = rows["rbits"].astype(np.int64)
    c = rows["count"].astype(np.int64)
    code = (c * (d - 1) * ab + 7) // 8 + (c * rb + 7) // 8
    ti = min(P, tile_geometry()[0])
    return PAGE_HEADER_BYTES + code + 2 * c * d_v, -(-c // ti)


# Planner cost model.  k_ada_decode is bound by the on-chip work per item
# (feature recurrence, LUT traffic), not by its bytes, and that work depends
# on the tier's angle width: measured per-item cost on a B200 (tools/
# tier_cost.py, profiles/r1*_tier_cost.log), in picoseconds per item at
# d = 128, one layer of 8 KV heads x 128K items.  Units are balanced on
# estimated time = items x cost(b_theta) (+ a small per-page term), so every
# CTA of a one-unit-per-CTA plan finishes together.
# (refined by a least-squares fit of per-CTA durations of mixed-tier c5
# launches, tools/cta_times.py: 9.95 / 14.4 / 17.6 / 24.2 ns per item per CTA
# for b_theta = 2 / 4 / 7 / 12 with the quad-row 2-bit tables -- same ratios,
# scaled to the single-tier runs)
PS_PER_ITEM = {1: 80, 2: 80, 3: 120, 4: 116, 5: 140, 6: 190, 7: 141, 8: 160, 9: 170, 10: 180,
               11: 190, 12: 195, 13: 400, 14: 430, 15: 470, 16: 500}
PAGE_COST_PS = 200
if os.environ.get("SPHKV_PS_PER_ITEM"):  # experiments: "2:80,4:116,..." overrides
    PS_PER_ITEM.update({int(a): int(b) for a, b in
                        (kv.split(":") for kv in os.environ["SPHKV_PS_PER_ITEM"].split(","))})


def _page_cost(rows, d):
    ab = rows["abits"].astype(np.int64)
    per = np.array([PS_PER_ITEM.get(int(b), 200) for b in range(17)], dtype=np.int64)[ab]
    scale = max(d - 1, 1) / 127.0  # work scales with the d-1 code rows
    return (rows["count"].astype(np.int64) * per * scale).astype(np.int64) + PAGE_COST_PS


def plan_store(store, groups=None, grid=SM_COUNT, units_per_cta=2, ranges=None,
               dynamic=False, tail=0.0, tail_pieces=2, open_end=False,
               open_reserve_tiles=0.0) -> DecodePlan:
    """Plan a decode pass over `groups` (default: every group of the store).

    `tail` (with units_per_cta=1, implies dynamic): each CTA's share is cut
    into one piece of (1 - tail) of it plus `tail_pieces` small pieces of the
    rest; CTAs claim the big pieces first, then the small ones as they
    finish, absorbing the per-CTA speed spread.

    `ranges` (optional, one (begin, end) per group) restricts each group to a
    contiguous range of its pointer list -- the page-range split of one
    sequence across ranks; see `plan_store_range`.

    `open_end`: each group's last unit runs to the list's current end (decode
    steps that append); with `open_reserve_tiles` (units_per_cta=1) that unit
    is cut that many average tiles short of an equal share, leaving room for
    the partly filled pages appends open (one per tier, each a whole tile)."""
    n, rows, plen, ptr = store._host()
    if groups is None:
        groups = np.arange(store.groups)
    groups = np.asarray(groups, dtype=np.int64)
    if ranges is None:
        ranges = [(0, int(plen[g])) for g in groups]
    pbytes, ptiles = _page_bytes(rows, store.tiers, store.d, store.d_v, store.page_size)
    pbytes = _page_cost(rows, store.d)  # balance on estimated time, not bytes
    lists = [ptr[g, rb:re] for g, (rb, re) in zip(groups, ranges)]
    total = sum(int(pbytes[l].sum()) for l in lists)
    target = max(total // max(grid * units_per_cta, 1), 1)
    pieces = []  # (bytes, group, begin, end, piece index)
    if units_per_cta == 1 and 0 < len(groups) <= grid and total > 0:
        grid_all = grid
        # one unit per CTA: give each group a share of the grid proportional
        # to its cost (largest remainder) and cut its list at the cost
        # quantiles, so every CTA gets ~total/grid and none gets two pieces
        gcost = np.array([int(pbytes[l].sum()) for l in lists], dtype=np.float64)
        grid = grid - int((gcost == 0).sum())  # empty groups keep a zero-cost slot of their own
        share = gcost / gcost.sum() * grid
        n_g = np.floor(share).astype(np.int64)
        n_g = np.where((gcost > 0) & (n_g == 0), 1, n_g)
        rem = grid - int(n_g.sum())
        for i in np.argsort(-(share - np.floor(share)), kind="stable")[:max(rem, 0)]:
            n_g[i] += 1
        while n_g.sum() > max(grid, int((gcost > 0).sum())):  # (the bumps to 1 can overshoot)
            n_g[int(np.argmax(n_g))] -= 1
        grid = grid_all
        for g, lst, (rb, _), n in zip(groups, lists, ranges, n_g):
            if len(lst) == 0:
                pieces.append([0, int(g), rb, rb])
                continue
            c = np.cumsum(pbytes[lst])
            # open-ended last unit: cut the list as if it carried
            # open_reserve_tiles more (average) tiles, which the last unit owns
            extra = 0.0
            if open_end and open_reserve_tiles > 0:
                extra = open_reserve_tiles * float(c[-1]) / max(int(ptiles[lst].sum()), 1)
            if tail > 0:
                ns = int(n) * int(tail_pieces)
                fr = [(1.0 - tail) * k / n for k in range(1, int(n) + 1)]
                fr += [(1.0 - tail) + tail * j / ns for j in range(1, ns)]
            else:
                fr = [k / n for k in range(1, int(n))]
            cuts = [0] + [int(np.searchsorted(c, (c[-1] + extra) * f, side="left")) + 1
                          for f in fr] + [len(lst)]
            cuts = np.minimum(np.maximum.accumulate(cuts), len(lst))
            for s0, e0 in zip(cuts[:-1], cuts[1:]):
                if e0 > s0:
                    while int(ptiles[lst[s0:e0]].sum()) > tile_geometry()[1]:  # tile cap
                        m = s0 + max(1, (e0 - s0) // 2)
                        pieces.append([int(pbytes[lst[s0:m]].sum()), int(g), rb + s0, rb + m])
                        s0 = m
                    pieces.append([int(pbytes[lst[s0:e0]].sum()), int(g), rb + s0, rb + e0])
        lists = []  # done
    for g, lst, (rb, _) in zip(groups, lists, ranges):
        b = pbytes[lst] if len(lst) else np.zeros(0, np.int64)
        t = ptiles[lst] if len(lst) else np.zeros(0, np.int64)
        start, acc, tacc = 0, 0, 0
        for k in range(len(lst)):
            if k > start and (acc + b[k] > target * 1.05 or tacc + t[k] > tile_geometry()[1]):
                pieces.append([acc, int(g), rb + start, rb + k])
                start, acc, tacc = k, 0, 0
            acc += int(b[k])
            tacc += int(t[k])
        pieces.append([acc, int(g), rb + start, rb + len(lst)])  # (possibly empty group)
    rng = {int(g): r for g, r in zip(groups, ranges)}
    dynamic = dynamic or (tail > 0 and units_per_cta == 1)
    if open_end:  # each group's last unit runs to the list's current end
        last = {}
        for pc in pieces:
            if pc[1] not in last or pc[2] >= last[pc[1]][2]:
                last[pc[1]] = pc
        for pc in last.values():
            pc[3] = -1
    return _finish(pieces, groups, grid,
                   lambda g: int(rows["count"][ptr[g, rng[g][0]:rng[g][1]]].sum()),
                   lambda g, s: int(rows["count"][ptr[g, rng[g][0]:s]].sum()) if s > rng[g][0]
                   else 0, dynamic)


def split_ranges(page_bytes, world):
    """Split one pointer list (per-page cost, pointer order) into
    `world` contiguous ranges balanced by cost, not page count (tiers differ
    in bytes per item).  Range r ends at the first page whose cumulative bytes
    reach (r+1)/world of the total; ranges may be empty."""
    b = np.asarray(page_bytes, dtype=np.int64)
    n = len(b)
    if n == 0:
        return [(0, 0)] * world
    c = np.cumsum(b)
    tot = int(c[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(c, tot * r / world, side="left")) + 1
                    if tot > 0 else (n * r) // world)
    cuts.append(n)
    cuts = np.minimum(np.maximum.accumulate(cuts), n)
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def rank_ranges(store, groups, rank, world):
    """This rank's pointer-list range of every group (page-range split)."""
    n, rows, plen, ptr = store._host()
    cost = _page_cost(rows, store.d)  # ranks balanced on estimated time
    return [split_ranges(cost[ptr[g, : plen[g]]], world)[rank] for g in groups]


def plan_store_range(store, groups, rank, world, grid=SM_COUNT, units_per_cta=2,
                     dynamic=False) -> DecodePlan:
    """Rank `rank`'s share of a page-range split of `groups` over `world` ranks.

    The rank's units cover only its ranges; `sphkv_lse_merge_ex(state_out=1)`
    turns its splits into one partial state per (group, q-head), those are
    all-gathered (rank-major) and merged again -- `merge_gathered`."""
    groups = np.asarray(groups, dtype=np.int64)
    return plan_store(store, groups, grid, units_per_cta,
                      ranges=rank_ranges(store, groups, rank, world), dynamic=dynamic)


def merge_local_state(plan, partials, G, d_v, state_out, stream=None):
    """Merge this rank's splits into one partial slot per planned group."""
    l = _lib.lib()
    _lib.check(l.sphkv_lse_merge_ex(partials.data_ptr(), plan.slot_begin.data_ptr(), 0, 0,
                                    len(plan.group_ids), G, d_v, state_out.data_ptr(), 1,
                                    _lib.stream_ptr(stream)))
    return state_out


def merge_gathered(n_groups, world, gathered, G, d_v, out, stream=None):
    """Merge the rank-major all-gather [world][n_groups] of per-rank states."""
    l = _lib.lib()
    _lib.check(l.sphkv_lse_merge_ex(gathered.data_ptr(), None, world, n_groups, n_groups, G,
                                    d_v, out.data_ptr(), 0, _lib.stream_ptr(stream)))
    return out


def plan_dense(dstore, groups=None, grid=SM_COUNT, units_per_cta=2, dynamic=False,
               pages=None) -> DecodePlan:
    """Dense baseline plan; `pages` = (first, end) restricts every group to a
    page range (sliding-window layers attend to their last pages only)."""
    G = dstore.batch * dstore.layers * dstore.heads
    if groups is None:
        groups = np.arange(G)
    groups = np.asarray(groups, dtype=np.int64)
    npg = dstore.n_pages_per_group
    p0, p1 = (0, npg) if pages is None else (max(0, int(pages[0])), min(npg, int(pages[1])))
    P = dstore.page_size
    per_page = PAGE_HEADER_BYTES + P * (dstore.d + dstore.d_v) * 2
    total = len(groups) * (p1 - p0) * per_page
    target = max(total // max(grid * units_per_cta, 1), 1)
    pages_per_unit = max(1, min(int(round(target / per_page)), MAX_UNIT_TILES * 64 // P))
    pieces = []
    for g in groups:
        for s in range(p0, max(p1, p0 + 1), pages_per_unit):
            e = min(p1, s + pages_per_unit)
            items = min(e * P, dstore.tokens) - s * P
            pieces.append([max(items, 0) * (dstore.d + dstore.d_v) * 2, int(g), s, e])
    T = dstore.tokens
    return _finish(pieces, groups, grid, lambda g: T,
                   lambda g, s: max(min(s * P, T), 0), dynamic)


def _finish(pieces, groups, grid, group_items_fn, piece_items_fn, dynamic=False):
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
    slot_group = np.array([order[p[1]] for p in pieces], dtype=np.int32)
    if dynamic:
        # CTAs claim units from a global queue in list order: longest first
        units, dbg = [], []
        for _, g, s, e, slot in sorted(pieces, key=lambda p: (-p[0], p[4])):
            units.append((g, s, e, slot))
            dbg.append(g_off[order[g]] + piece_items_fn(g, s))
        arr = np.array(units, dtype=np.int32).reshape(-1, 4)
        u = np.zeros(len(arr), dtype=_lib.UNIT_DTYPE)
        u["group"], u["ptr_begin"], u["ptr_end"], u["out_slot"] = arr.T
        return DecodePlan(u, slot_begin, n_slots, max(1, min(grid, len(pieces))), gi_items,
                          groups, np.asarray(dbg, dtype=np.int64), slot_group, True)
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
                dbg.append(g_off[order[g]] + piece_items_fn(g, s))
            else:
                units.append((int(groups[0]) if len(groups) else 0, 0, 0, scratch))
                dbg.append(0)
    arr = np.array(units, dtype=np.int32).reshape(-1, 4)
    u = np.zeros(len(arr), dtype=_lib.UNIT_DTYPE)
    u["group"], u["ptr_begin"], u["ptr_end"], u["out_slot"] = arr.T
    return DecodePlan(u, slot_begin, n_slots, grid, gi_items, groups,
                      np.asarray(dbg, dtype=np.int64), slot_group, False)
