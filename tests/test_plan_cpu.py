"""Planner host logic on CPU (no device): the one-unit-per-CTA balanced split
(SURVEY 7.3 item 5), the greedy multi-unit split, slot layout for the fused
merge, debug-logit offsets, and the page-range split across ranks."""

import numpy as np

from paper_2605_18856_b200 import _lib, plan as planmod
from paper_2605_18856_b200.codec import TierSpec, TierTable


class FakeStore:
    """Just what the planner reads: page table rows and pointer lists."""

    def __init__(self, counts_by_group, abits_by_group, P=256, d=128):
        self.page_size, self.d, self.d_v = P, d, d
        self.tiers = TierTable((TierSpec(0, 0, 0, 0), TierSpec(1, 2, 4, 8), TierSpec(2, 12, 14, 8)))
        rows, lists = [], []
        for counts, bits in zip(counts_by_group, abits_by_group):
            lst = []
            for c, b in zip(counts, bits):
                lst.append(len(rows))
                rows.append((c, b))
            lists.append(lst)
        self.groups = len(lists)
        r = np.zeros(len(rows), dtype=_lib.PAGE_DTYPE)
        r["count"] = [c for c, _ in rows]
        r["abits"] = [b for _, b in rows]
        r["rbits"] = 8
        cap = max(len(l) for l in lists)
        ptr = np.zeros((self.groups, cap), dtype=np.int32)
        plen = np.array([len(l) for l in lists], dtype=np.int32)
        for g, l in enumerate(lists):
            ptr[g, : len(l)] = l
        self._h = (len(rows), r, plen, ptr)

    def _host(self):
        return self._h


def make_store(seed=0, groups=8, pages=400):
    rng = np.random.default_rng(seed)
    counts, bits = [], []
    for _ in range(groups):
        n = rng.integers(pages // 2, pages)
        c = np.full(n, 256)
        c[rng.integers(0, n, 3)] = rng.integers(1, 256, 3)  # partial pages
        b = np.sort(rng.choice([2, 12], n, p=[0.7, 0.3]))    # tier ascending
        counts.append(c)
        bits.append(b)
    counts.append(np.zeros(0, int))  # an empty group
    bits.append(np.zeros(0, int))
    return FakeStore(counts, bits)


def unit_cost(st, plan):
    n, rows, plen, ptr = st._host()
    cost = planmod._page_cost(rows, st.d)
    u = plan.units_host
    return np.array([cost[ptr[g, a:b]].sum() for g, a, b in zip(u["group"], u["ptr_begin"],
                                                                u["ptr_end"])])


def check_cover(st, plan):
    """every page of every planned group in exactly one unit; slots contiguous per group"""
    n, rows, plen, ptr = st._host()
    u = plan.units_host
    seen = {}
    for g, a, b, slot in zip(u["group"], u["ptr_begin"], u["ptr_end"], u["out_slot"]):
        if slot == plan.n_slots:
            continue  # padding unit
        for pos in range(a, b):
            assert (g, pos) not in seen
            seen[(g, pos)] = slot
        gi = list(plan.group_ids).index(g)
        assert plan.slot_begin_host[gi] <= slot < plan.slot_begin_host[gi + 1]
    for g in plan.group_ids:
        for pos in range(plen[g]):
            assert (g, pos) in seen
    assert plan.slot_begin_host[-1] == plan.n_slots


def test_balanced_one_unit_per_cta():
    st = make_store()
    plan = planmod.plan_store(st, grid=148, units_per_cta=1)
    check_cover(st, plan)
    assert plan.n_units <= 148
    c = unit_cost(st, plan)
    c = c[c > 0]
    # equal shares up to page granularity (one 12-bit page ~ 1/20 of a share here)
    n, rows, plen, ptr = st._host()
    page_max = planmod._page_cost(rows, st.d).max()
    assert c.max() <= c.mean() + 2 * page_max


def test_greedy_multi_unit_and_dynamic_order():
    st = make_store(1)
    for dyn in (False, True):
        plan = planmod.plan_store(st, grid=16, units_per_cta=3, dynamic=dyn)
        check_cover(st, plan)
        if dyn:  # claimed longest first
            c = unit_cost(st, plan)
            assert np.all(np.diff(c) <= 0)


def test_rank_ranges_partition_groups():
    st = make_store(2)
    groups = list(range(st.groups))
    world = 3
    per_rank = [planmod.rank_ranges(st, groups, r, world) for r in range(world)]
    n, rows, plen, ptr = st._host()
    for gi, g in enumerate(groups):
        spans = [per_rank[r][gi] for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == plen[g]
        for (a, b), (c, d) in zip(spans[:-1], spans[1:]):
            assert b == c
    for r in range(world):
        plan = planmod.plan_store_range(st, groups, r, world, grid=8)
        u = plan.units_host
        for g, a, b, slot in zip(u["group"], u["ptr_begin"], u["ptr_end"], u["out_slot"]):
            if slot == plan.n_slots:
                continue  # padding unit (empty range, scratch slot)
            lo, hi = per_rank[r][groups.index(g)]
            assert lo <= a <= b <= hi


def test_tail_pieces_claimed_after_the_big_ones():
    """tail > 0: one big piece per CTA share first in the claim order, then
    the small pieces; every page covered exactly once."""
    st = make_store()
    plan = planmod.plan_store(st, grid=148, units_per_cta=1, tail=0.2, tail_pieces=2)
    check_cover(st, plan)
    assert plan.dynamic
    c = unit_cost(st, plan)
    nz = c[c > 0]
    assert len(nz) > 148
    big = np.sort(nz)[::-1][:min(148, len(nz) // 3)]
    assert np.all(c[: len(big)] >= np.sort(c[len(big):]).max() * 0.99)
