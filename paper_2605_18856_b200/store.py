"""Device-resident paged KV store (drop-in for sphkv.store, pkg/src/sphkv/store.py).

`PagedStore` keeps every page in HBM in the B200 page format described in
include/sphkv_b200.h: a code pool (per page the word-interleaved item-major
angle block -- each item's code string cut into 16-byte quads interleaved
across 32-item granules -- then the radius row), an fp16 value pool with
16-byte swizzled rows, and a page table / pointer lists.  Packing, appending and exporting run
as sm_100a kernels; the host keeps only the reference's accounting model
(TrafficMeter, ResidentBreakdown -- closed-form byte counts, store.py:51-133)
and lazily materialized page views for inspection.

Reference-format byte streams (Page.angle_stream / radius_stream, SPHKV1
snapshots) are produced by the `sphkv_export_streams` kernel, which re-strides
partial pages; tests assert them byte-identical to the reference.
"""

from __future__ import annotations

import ctypes
import struct
import threading
from dataclasses import dataclass

import numpy as np

from . import _lib
from .codec import DROP_TIER_ID, SphericalKey, TierSpec, TierTable

PAGE_HEADER_BYTES = 16
PTR_ENTRY_BYTES = 8
VALUE_BYTES_PER_ENTRY = 2
FILE_MAGIC = b"SPHKV1"
FILE_DIRECTORY_BYTES = len(FILE_MAGIC) + 24
METER_CATEGORIES = ("header", "k_codes", "values", "dense_k_write", "dense_k_read")
APPEND_SCALE_HEADROOM = 1.25


def packed_nbytes(count: int, bits: int) -> int:
    return (count * bits + 7) // 8


class TrafficMeter:
    """Deterministic byte meter (store.py:51-111): the reference's accounting
    model, kept host-side next to the real ncu DRAM counters."""

    def __init__(self):
        self._lock = threading.Lock()
        self.reset()

    def reset(self):
        with getattr(self, "_lock", threading.Lock()):
            self.read_bytes = 0
            self.write_bytes = 0
            self.decode_tokens = 0
            self.category = {c: 0 for c in METER_CATEGORIES}

    def add_read(self, category, nbytes):
        with self._lock:
            self.read_bytes += int(nbytes)
            self.category[category] += int(nbytes)

    def add_write(self, category, nbytes):
        with self._lock:
            self.write_bytes += int(nbytes)
            self.category[category] += int(nbytes)

    def add_batch(self, reads=(), writes=()):
        with self._lock:
            for cat, n in reads:
                self.read_bytes += int(n)
                self.category[cat] += int(n)
            for cat, n in writes:
                self.write_bytes += int(n)
                self.category[cat] += int(n)

    def tick(self, n=1):
        with self._lock:
            self.decode_tokens += n

    @property
    def total_bytes(self):
        return self.read_bytes + self.write_bytes

    def b_hbm(self):
        return None if self.decode_tokens == 0 else self.total_bytes / self.decode_tokens

    def snapshot(self):
        with self._lock:
            snap = dict(self.category)
            snap.update(read_bytes=self.read_bytes, write_bytes=self.write_bytes,
                        decode_tokens=self.decode_tokens)
        return snap


@dataclass
class ResidentBreakdown:
    payload_bytes: int = 0
    header_bytes: int = 0
    ptr_bytes: int = 0
    tag_bytes: int = 0
    prot_bytes: int = 0
    frag_bytes: int = 0

    @property
    def total(self) -> int:
        return (self.payload_bytes + self.header_bytes + self.ptr_bytes + self.tag_bytes
                + self.prot_bytes + self.frag_bytes)

    @property
    def eta_meta(self) -> float:
        return 0.0 if self.total == 0 else (self.total - self.payload_bytes) / self.total


def _page_formulas(count, capacity, tier: TierSpec, d, d_v):
    """Per-page byte formulas (store.py:178-203)."""
    ang = packed_nbytes(count * (d - 1), tier.angle_bits)
    rad = packed_nbytes(count, tier.radius_bits)
    val = count * d_v * VALUE_BYTES_PER_ENTRY
    tag = (count * tier.meta_bits + 7) // 8
    prot = (count + 7) // 8
    key_bits = (d - 1) * tier.angle_bits + tier.radius_bits + tier.meta_bits
    slot = (key_bits + 7) // 8 + d_v * VALUE_BYTES_PER_ENTRY
    return ang, rad, val, tag, prot, (capacity - count) * slot


def code_block_bytes(d, P, abits, rbits):
    """Device code block of one page (word-interleaved angle part + radius
    row, see include/sphkv_b200.h); mirrors common.cuh:code_block_bytes."""
    words = (((d - 1) * abits + 31) // 32 + 3) // 4 * 4
    angle = (P + 31) // 32 * words * 128
    rbytes = (P * rbits + 7) // 8
    return angle + (rbytes + 15) // 16 * 16


class PageView:
    """Host view of one device page with the reference Page interface."""

    __slots__ = ("_store", "index", "tier", "layer", "head", "seq", "capacity", "count",
                 "radius_scale", "_streams")

    def __init__(self, store, index, row):
        self._store = store
        self.index = index
        self.tier = store.tiers.spec_for(int(row["tier"]))
        g = int(row["group"])
        self.head = g % store.heads
        self.layer = (g // store.heads) % store.layers
        self.seq = g // (store.heads * store.layers)
        self.capacity = store.page_size
        self.count = int(row["count"])
        self.radius_scale = float(row["radius_scale"])
        self._streams = None

    @property
    def full(self):
        return self.count >= self.capacity

    def _get(self):
        if self._streams is None:
            self._streams = self._store._export_page(self.index)
        return self._streams

    def angle_stream_bytes(self, d):
        return packed_nbytes(self.count * (d - 1), self.tier.angle_bits)

    def radius_stream_bytes(self):
        return packed_nbytes(self.count, self.tier.radius_bits)

    def value_block_bytes(self, d_v):
        return self.count * d_v * VALUE_BYTES_PER_ENTRY

    def payload_bytes(self, d, d_v):
        return self.angle_stream_bytes(d) + self.radius_stream_bytes() + self.value_block_bytes(d_v)

    def tag_bytes(self):
        return (self.count * self.tier.meta_bits + 7) // 8

    def prot_bytes(self):
        return (self.count + 7) // 8

    def slot_bytes(self, d, d_v):
        kb = (d - 1) * self.tier.angle_bits + self.tier.radius_bits + self.tier.meta_bits
        return (kb + 7) // 8 + d_v * VALUE_BYTES_PER_ENTRY

    def frag_bytes(self, d, d_v):
        return (self.capacity - self.count) * self.slot_bytes(d, d_v)

    def angle_stream(self, d=None):
        return self._get()["angle"]

    def radius_stream(self):
        return self._get()["radius"]

    @property
    def values(self):
        return self._get()["values"].astype(np.float64)

    @property
    def protect(self):
        return self._get()["protect"].astype(bool)

    @property
    def token_ids(self):
        return self._store._token_ids(self.index, self.count)

    @property
    def angle_codes(self):
        from .bitpack import unpack_bits

        d = self._store.d
        soa = unpack_bits(self.angle_stream(), self.tier.angle_bits, self.count * (d - 1))
        return soa.reshape(d - 1, self.count).T.copy()

    @property
    def radius_codes(self):
        from .bitpack import unpack_bits

        return unpack_bits(self.radius_stream(), self.tier.radius_bits, self.count)


class PagedStore:
    """Paged, tier-homogeneous store in HBM (store.py:214-427).

    Extra keyword arguments size the device pools: `batch` sequences share
    one store (groups = batch*layers*heads), `capacity_tokens` bounds the
    items per group, `append_tokens` reserves decode-time appends."""

    def __init__(self, tiers: TierTable, layers: int, heads: int, d: int, d_v: int,
                 page_size: int, meter: TrafficMeter | None = None, *, batch: int = 1,
                 capacity_tokens: int = 1024, append_tokens: int = 256,
                 max_pages: int | None = None, code_bytes: int | None = None):
        import torch

        if page_size < 1:
            raise ValueError("page size must be >= 1")
        tiers.validate_rates(d)
        if page_size % 32 != 0:
            raise ValueError(f"device page_size must be a multiple of 32, got {page_size}")
        for t in tiers.non_drop:
            if t.angle_bits > 16 or t.radius_bits > 16:
                raise ValueError(f"tier {t.id}: device codes support at most 16 bits")
        if len(tiers.tiers) > _lib.MAX_TIERS:
            raise ValueError("at most 16 tiers")
        self.tiers = tiers
        self.batch, self.layers, self.heads = batch, layers, heads
        self.d, self.d_v, self.page_size = d, d_v, page_size
        self.dvp = (d_v + 15) // 16 * 16
        self.meter = meter if meter is not None else TrafficMeter()
        self.groups = batch * layers * heads
        ntiers = len(tiers.non_drop)
        per_group = -(-(capacity_tokens + append_tokens) // page_size) + ntiers + 2
        self.max_pages = max(self.groups * per_group, 1)
        self.ptr_cap = per_group + 8
        max_block = max(code_block_bytes(d, page_size, t.angle_bits, t.radius_bits)
                        for t in tiers.non_drop)
        self.code_cap = self.max_pages * max_block + 256
        # explicit pool sizes (a caller that knows the allocation, e.g. the
        # benchmark: the worst case -- every item at the widest tier -- does
        # not fit a 128K-token batch in HBM)
        if max_pages is not None:
            self.max_pages = max(int(max_pages), 1)
        if code_bytes is not None:
            self.code_cap = int(code_bytes) + 256
        dev = "cuda"
        self.t_pages = torch.zeros(self.max_pages * 32, dtype=torch.uint8, device=dev)
        self.t_ptr = torch.zeros(self.groups * self.ptr_cap, dtype=torch.int32, device=dev)
        self.t_ptr_len = torch.zeros(self.groups, dtype=torch.int32, device=dev)
        self.t_group_last = torch.full((self.groups * _lib.MAX_TIERS,), -1, dtype=torch.int32,
                                       device=dev)
        # tail slack: the decode look-ahead may read a few rows past the last block
        self.t_codes = torch.zeros(self.code_cap + 16384, dtype=torch.uint8, device=dev)
        self.t_values = torch.zeros(self.max_pages * page_size * self.dvp, dtype=torch.float16,
                                    device=dev)
        self.t_protect = torch.zeros(self.max_pages * page_size, dtype=torch.uint8, device=dev)
        self.t_token_ids = torch.full((self.max_pages * page_size,), -1, dtype=torch.int64,
                                      device=dev)
        self.t_counters = torch.zeros(4, dtype=torch.int64, device=dev)
        self.t_lut = None
        self._host_cache = None
        self._rebuild_cstruct()

    # -- C struct ------------------------------------------------------------
    def _rebuild_cstruct(self):
        old = getattr(self, "cstruct", None)
        c = _lib.CStore()
        if old is not None:  # keep the table placement hint across pool growth
            for k in range(_lib.MAX_TIERS):
                c.lut_items[k] = old.lut_items[k]
            c.lut_flags = old.lut_flags
        c.batch, c.layers, c.heads = self.batch, self.layers, self.heads
        c.d, c.d_v, c.page_size = self.d, self.d_v, self.page_size
        c.n_tiers = len(self.tiers.tiers)
        c.max_pages, c.ptr_cap, c.code_cap = self.max_pages, self.ptr_cap, self.code_cap
        c.tiers = _lib.tiers_to_c(self.tiers)
        c.pages = self.t_pages.data_ptr()
        c.ptr = self.t_ptr.data_ptr()
        c.ptr_len = self.t_ptr_len.data_ptr()
        c.group_last = self.t_group_last.data_ptr()
        c.codes = self.t_codes.data_ptr()
        c.values = self.t_values.data_ptr()
        c.protect = self.t_protect.data_ptr()
        c.token_ids = self.t_token_ids.data_ptr()
        c.counters = self.t_counters.data_ptr()
        self.cstruct = c
        self._build_lut()

    def _refresh_lut(self):
        """Place the shared-memory tables by the tiers actually stored (items
        per tier index as the layout hint: absent tiers get no table, the most
        used tiers are replicated first) and rebuild them when that changes."""
        n, rows, _, _ = self._host()
        ids = [t.id for t in self.tiers.tiers]
        items = [0] * _lib.MAX_TIERS
        if n:
            for k, tid in enumerate(ids):
                items[k] = int(rows["count"][rows["tier"] == tid].sum())
        if list(self.cstruct.lut_items) != items:
            for k in range(_lib.MAX_TIERS):
                self.cstruct.lut_items[k] = items[k]
            self._build_lut()

    def _build_lut(self):
        """(Re)build the prebuilt shared-memory tables for the current layout
        hint and lut_flags; both variants (with / without the 2-bit table)
        are cached so launches with different GQA widths do not rebuild."""
        import torch

        l = _lib.require_gpu()
        c = self.cstruct
        c.tiers = _lib.tiers_to_c(self.tiers)
        key = (int(c.lut_flags), tuple(c.lut_items))
        cache = self.__dict__.setdefault("_lut_cache", {})
        if key in cache and cache[key][2] == self._lut_gen():
            t, off, _ = cache[key]
            c.lut = t.data_ptr()
            for k in range(_lib.MAX_TIERS):
                c.lut_off[k] = off[k]
            return
        n = l.sphkv_lut_floats(ctypes.byref(c))
        t = torch.zeros(n, dtype=torch.float32, device="cuda")
        c.lut = t.data_ptr()
        _lib.check(l.sphkv_store_build_lut(ctypes.byref(c), _lib.stream_ptr()))
        cache[key] = (t, tuple(c.lut_off), self._lut_gen())
        self.t_lut = t

    def _lut_gen(self):
        # the tables depend only on the tier widths (eps changes do not matter)
        return tuple((t.id, t.angle_bits) for t in self.tiers.tiers)

    # Decode the 2-bit tier from per-query h-byte tables (csrc/hb_tile.cuh,
    # exact; 3x fewer instructions per 2-bit item) instead of the quad-row
    # table.  Off by default: measured no faster end to end on c5 (the decode
    # is bound by per-tile latency and the P.V / V-ring pipeline, not by the
    # 2-bit tier's instruction count -- DESIGN.md section 4).
    hbyte_tables = False

    def uses_hb(self, G):
        """Launches with G query heads decode the 2-bit tier from per-query
        h-byte tables (csrc/hb_tile.cuh) instead of the quad-row table."""
        return (self.hbyte_tables and G <= 4 and self.d in (64, 128)
                and self.page_size % 128 == 0
                and any(t.angle_bits == 2 for t in self.tiers.non_drop))

    def cptr_for(self, G):
        """C struct for a decode launch with G query heads: selects (building
        once) the prebuilt table variant that launch mode uses."""
        hb = 1 if self.uses_hb(G) else 0
        if self.cstruct.lut_flags != hb:
            self.cstruct.lut_flags = hb
            self._build_lut()
        return self.cptr

    @property
    def cptr(self):
        self.cstruct.tiers = _lib.tiers_to_c(self.tiers)  # eps may be calibrated later
        return ctypes.byref(self.cstruct)

    def _invalidate(self):
        self._host_cache = None

    def _host(self):
        """Download page table + pointer lists (cached until the next mutation)."""
        if self._host_cache is None:
            n = int(self.t_counters[0].item())
            pages = self.t_pages[: n * 32].cpu().numpy().view(_lib.PAGE_DTYPE)
            plen = self.t_ptr_len.cpu().numpy()
            ptr = self.t_ptr.cpu().numpy().reshape(self.groups, self.ptr_cap)
            self._host_cache = (n, pages, plen, ptr)
        return self._host_cache

    @property
    def n_pages(self) -> int:
        return self._host()[0]

    # -- reference-shaped views -----------------------------------------------
    def _group(self, layer, head, seq=0):
        return (seq * self.layers + layer) * self.heads + head

    @property
    def pages(self):
        n, rows, _, _ = self._host()
        return [PageView(self, i, rows[i]) for i in range(n)]

    @property
    def pointer(self):
        _, _, plen, ptr = self._host()
        out = {}
        for l in range(self.layers):
            for h in range(self.heads):
                g = self._group(l, h)
                out[(l, h)] = [int(x) for x in ptr[g, : plen[g]]]
        return out

    def group_pages(self, g):
        _, _, plen, ptr = self._host()
        return ptr[g, : plen[g]]

    def _export_all(self):
        """Run the export kernel for every page; returns per-page dicts."""
        import torch

        n, rows, _, _ = self._host()
        if n == 0:
            return []
        d, dv = self.d, self.d_v
        sizes = []
        for r in rows:
            t = self.tiers.spec_for(int(r["tier"]))
            c = int(r["count"])
            a = packed_nbytes(c * (d - 1), t.angle_bits)
            b = packed_nbytes(c, t.radius_bits)
            sizes.append((a, b, 2 * c * dv, c))
        offs = np.zeros(n + 1, dtype=np.int64)
        offs[1:] = np.cumsum([sum(s) for s in sizes])
        out = torch.zeros(int(offs[-1]) + 16, dtype=torch.uint8, device="cuda")
        offs_d = torch.as_tensor(offs[:-1], device="cuda")
        l = _lib.require_gpu()
        _lib.check(l.sphkv_export_streams(self.cptr, n, offs_d.data_ptr(), out.data_ptr(),
                                          _lib.stream_ptr()))
        blob = out.cpu().numpy()
        res = []
        for i, (a, b, v, c) in enumerate(sizes):
            o = int(offs[i])
            res.append({
                "angle": blob[o: o + a].copy(),
                "radius": blob[o + a: o + a + b].copy(),
                "values": blob[o + a + b: o + a + b + v].view(np.float16).reshape(c, dv).copy(),
                "protect": blob[o + a + b + v: o + a + b + v + c].copy(),
            })
        return res

    def _export_page(self, idx):
        cache = getattr(self, "_export_cache", None)
        if cache is None or cache[0] is not self._host_cache:
            self._export_cache = (self._host_cache, self._export_all())
        return self._export_cache[1][idx]

    def _token_ids(self, idx, count):
        P = self.page_size
        return self.t_token_ids[idx * P: idx * P + count].cpu().numpy()

    # -- construction ----------------------------------------------------------
    def append_item(self, layer, head, key: SphericalKey, value, tier_id, protected=False,
                    token_id=-1, meter_write=True):
        """Append one coded state (store.py:249-274) through the device append kernel."""
        if tier_id == DROP_TIER_ID:
            return
        tier = self.tiers.spec_for(tier_id)
        if (layer, head) not in {(l, h) for l in range(self.layers) for h in range(self.heads)}:
            raise KeyError(f"unknown (layer, head) = {(layer, head)}")
        g = self._group(layer, head)
        n = self.groups
        tid = np.zeros(n, dtype=np.int16)
        tid[g] = tier_id
        active = np.zeros(n, dtype=np.uint8)
        active[g] = 1
        radii = np.zeros(n)
        radii[g] = key.radius
        ang = np.zeros((n, self.d - 1))
        ang[g] = key.angles
        vals = np.zeros((n, self.d_v), dtype=np.float16)
        vals[g] = np.asarray(value, dtype=np.float64).astype(np.float16)
        prot = np.zeros(n, dtype=np.uint8)
        prot[g] = bool(protected)
        toks = np.full(n, -1, dtype=np.int64)
        toks[g] = token_id
        before = self.n_pages
        self.append_batch(radii=radii, angles=ang, values=vals, tier_ids=tid, protect=prot,
                          token_ids=toks, active=active)
        if meter_write:
            if self.n_pages > before:
                self.meter.add_write("header", PAGE_HEADER_BYTES + PTR_ENTRY_BYTES)
            kb = packed_nbytes(self.d - 1, tier.angle_bits) + packed_nbytes(1, tier.radius_bits)
            self.meter.add_write("k_codes", kb)
            self.meter.add_write("values", self.d_v * VALUE_BYTES_PER_ENTRY)

    def append_batch(self, *, keys=None, key_dtype=None, radii=None, angles=None, values,
                     tier_ids, protect=None, token_ids=None, active=None):
        """One appended state per group (device tensors or numpy arrays)."""
        import torch

        l = _lib.require_gpu()

        def dev(x, dt):
            if x is None:
                return None
            if isinstance(x, torch.Tensor):
                return x.to(device="cuda", dtype=dt).contiguous()
            return torch.as_tensor(np.ascontiguousarray(x), device="cuda").to(dt)

        n = self.groups
        ws = torch.empty(l.sphkv_append_workspace_bytes(n), dtype=torch.uint8, device="cuda")
        k = dev(keys, key_dtype or torch.float64) if keys is not None else None
        kd = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
              torch.float16: _lib.F16}[k.dtype] if k is not None else 0
        r = dev(radii, torch.float64)
        a = dev(angles, torch.float64)
        v = _lib.to_f16(values)
        t = dev(tier_ids, torch.int16)
        p = dev(protect, torch.uint8)
        tk = dev(token_ids, torch.int64)
        ac = dev(active, torch.uint8)
        self._ensure_append_capacity()
        _lib.check(l.sphkv_append(self.cptr, _lib.ptr(k), kd, _lib.ptr(r), _lib.ptr(a),
                                  _lib.ptr(v), _lib.ptr(t), _lib.ptr(p), _lib.ptr(tk),
                                  _lib.ptr(ac), ws.data_ptr(), _lib.stream_ptr()))
        err = int(ws[:4].view(torch.int32).item())
        self._invalidate()
        if err == 0:  # a tier's first pages may have opened: give it a table
            sel = t if ac is None else t[ac.bool()]
            ids = [t_.id for t_ in self.tiers.tiers]
            new = [int(x) for x in torch.unique(sel).cpu().tolist() if int(x) != DROP_TIER_ID]
            if any(self.cstruct.lut_items[ids.index(x)] == 0 for x in new if x in ids):
                self._refresh_lut()
        if err == 3:
            raise RuntimeError("store pool exhausted")
        if err == 4:
            raise RuntimeError("pointer list capacity exceeded")
        if err == 5:
            raise KeyError("unknown tier id in append")

    def _ensure_append_capacity(self):
        n = int(self.t_counters[0].item())
        used = int(self.t_counters[1].item())
        max_block = max(code_block_bytes(self.d, self.page_size, t.angle_bits, t.radius_bits)
                        for t in self.tiers.non_drop)
        if n + self.groups > self.max_pages or used + self.groups * max_block > self.code_cap:
            self._grow(2 * self.max_pages)
        _, _, plen, _ = self._host()
        if plen.size and int(plen.max()) + 1 > self.ptr_cap:
            self._grow(self.max_pages, ptr_cap=2 * self.ptr_cap)

    def _grow(self, max_pages, ptr_cap=None):
        import torch

        P, dvp = self.page_size, self.dvp
        max_block = max(code_block_bytes(self.d, P, t.angle_bits, t.radius_bits)
                        for t in self.tiers.non_drop)

        def extend(t, n, fill=0):
            out = torch.full((n,), fill, dtype=t.dtype, device=t.device)
            out[: t.numel()] = t
            return out

        self.t_pages = extend(self.t_pages, max_pages * 32)
        self.t_codes = extend(self.t_codes, max_pages * max_block + 256 + 16384)
        self.t_values = extend(self.t_values, max_pages * P * dvp)
        self.t_protect = extend(self.t_protect, max_pages * P)
        self.t_token_ids = extend(self.t_token_ids, max_pages * P, -1)
        self.max_pages = max_pages
        self.code_cap = max_pages * max_block + 256
        if ptr_cap is not None and ptr_cap > self.ptr_cap:
            old = self.t_ptr.view(self.groups, self.ptr_cap)
            new = torch.zeros((self.groups, ptr_cap), dtype=torch.int32, device="cuda")
            new[:, : self.ptr_cap] = old
            self.t_ptr = new.view(-1)
            self.ptr_cap = ptr_cap
        self._rebuild_cstruct()
        self._invalidate()

    def set_protect(self, page_idx, slot, flag):
        self.t_protect[page_idx * self.page_size + slot] = int(bool(flag))
        self._invalidate()
        self.meter.add_write("header", 1)

    # -- streaming / accounting ----------------------------------------------
    def stream_pages(self, layer, head, metered=True):
        if not (0 <= layer < self.layers and 0 <= head < self.heads):
            raise KeyError(f"unknown (layer, head) = {(layer, head)}")
        n, rows, _, _ = self._host()
        for idx in self.group_pages(self._group(layer, head)):
            page = PageView(self, int(idx), rows[int(idx)])
            if metered:
                self.meter.add_read("header", PAGE_HEADER_BYTES)
                self.meter.add_read("k_codes", page.angle_stream_bytes(self.d)
                                    + page.radius_stream_bytes())
                self.meter.add_read("values", page.value_block_bytes(self.d_v))
            yield int(idx), page

    def stream_head(self, layer, head, metered=True):
        from .codec import AngleCode

        for _, page in self.stream_pages(layer, head, metered=metered):
            levels = float((1 << page.tier.radius_bits) - 1)
            radii = page.radius_codes.astype(np.float64) / levels * page.radius_scale
            codes = page.angle_codes
            vals = page.values
            prot = page.protect
            for j in range(page.count):
                yield (page.tier.id, float(radii[j]), AngleCode(codes[j].copy()), vals[j],
                       bool(prot[j]))

    def meter_stream(self, layer, head, seq=0):
        """Meter one streamed pass over a head's pages in one batched call
        (totals identical to stream_pages' per-page reads, decode.py:336-342)."""
        if not (0 <= layer < self.layers and 0 <= head < self.heads):
            raise KeyError(f"unknown (layer, head) = {(layer, head)}")
        n, rows, _, _ = self._host()
        hdr = code = val = 0
        for idx in self.group_pages(self._group(layer, head, seq)):
            r = rows[int(idx)]
            t = self.tiers.spec_for(int(r["tier"]))
            a, b, v, *_ = _page_formulas(int(r["count"]), self.page_size, t, self.d, self.d_v)
            hdr += PAGE_HEADER_BYTES
            code += a + b
            val += v
        self.meter.add_batch((("header", hdr), ("k_codes", code), ("values", val)))

    def retained_count(self, layer=None, head=None):
        n, rows, _, _ = self._host()
        total = 0
        for r in rows:
            g = int(r["group"])
            h, l = g % self.heads, (g // self.heads) % self.layers
            if (layer is None or l == layer) and (head is None or h == head):
                total += int(r["count"])
        return total

    def expected_stream_bytes(self, layer, head, seq=0):
        n, rows, _, _ = self._host()
        total = 0
        for idx in self.group_pages(self._group(layer, head, seq)):
            r = rows[int(idx)]
            t = self.tiers.spec_for(int(r["tier"]))
            a, b, v, *_ = _page_formulas(int(r["count"]), self.page_size, t, self.d, self.d_v)
            total += PAGE_HEADER_BYTES + a + b + v
        return total

    def stream_bytes_total(self):
        """Algorithmic decode bytes of one full pass over every group (8(d)):
        per page header + packed code streams + fp16 values (store.py:315-322)."""
        n, rows, _, _ = self._host()
        c = rows["count"].astype(np.int64)
        a = (c * (self.d - 1) * rows["abits"].astype(np.int64) + 7) // 8
        b = (c * rows["rbits"].astype(np.int64) + 7) // 8
        return int(PAGE_HEADER_BYTES * n + a.sum() + b.sum() + (c * self.d_v * 2).sum())

    def resident_breakdown(self) -> ResidentBreakdown:
        n, rows, _, _ = self._host()
        br = ResidentBreakdown()
        for r in rows:
            t = self.tiers.spec_for(int(r["tier"]))
            a, b, v, tag, prot, frag = _page_formulas(int(r["count"]), self.page_size, t,
                                                      self.d, self.d_v)
            br.payload_bytes += a + b + v
            br.tag_bytes += tag
            br.prot_bytes += prot
            br.frag_bytes += frag
        br.header_bytes = PAGE_HEADER_BYTES * n
        br.ptr_bytes = FILE_DIRECTORY_BYTES + PTR_ENTRY_BYTES * (self.groups + n)
        return br

    def b_kv(self, t_active):
        if t_active < 1:
            raise ValueError("T_active must be >= 1")
        return self.resident_breakdown().total / t_active

    def check_invariants(self):
        """Tier homogeneity, scale bound, pointer coverage (store.py:343-358)."""
        n, rows, plen, ptr = self._host()
        seen = set()
        for g in range(self.groups):
            for idx in ptr[g, : plen[g]]:
                idx = int(idx)
                assert idx not in seen, "page listed twice"
                seen.add(idx)
                assert int(rows[idx]["group"]) == g
                assert int(rows[idx]["count"]) <= self.page_size
        assert len(seen) == n, "orphan pages outside pointer table"
        for p in self.pages:
            if p.count:
                levels = float((1 << p.tier.radius_bits) - 1)
                radii = p.radius_codes.astype(np.float64) / levels * p.radius_scale
                assert radii.max() <= p.radius_scale * (1 + 1e-9)

    # -- snapshot --------------------------------------------------------------
    def to_bytes(self) -> bytes:
        """SPHKV1 snapshot bytes (store.py:362-388) from device pages."""
        if self.batch != 1:
            raise ValueError("SPHKV1 snapshots hold one sequence (batch=1)")
        n, rows, plen, ptr = self._host()
        ex = self._export_all()
        parts = [FILE_MAGIC, struct.pack("<6I", self.layers, self.heads, self.d, self.d_v,
                                         self.page_size, n)]
        for i in range(n):
            r = rows[i]
            t = self.tiers.spec_for(int(r["tier"]))
            g = int(r["group"])
            c = int(r["count"])
            parts.append(struct.pack("<BBBBId", t.id, (g // self.heads) % self.layers,
                                     g % self.heads, 0, c, float(r["radius_scale"])))
            parts.append(np.packbits(ex[i]["protect"].astype(bool)).tobytes())
            parts.append(b"\x00" * ((c * t.meta_bits + 7) // 8))
            parts.append(ex[i]["angle"].tobytes())
            parts.append(ex[i]["radius"].tobytes())
            parts.append(ex[i]["values"].tobytes())
        for g in range(self.groups):
            idxs = ptr[g, : plen[g]].astype(np.uint64)
            parts.append(struct.pack("<Q", len(idxs)))
            parts.append(idxs.tobytes())
        return b"".join(parts)

    def to_file(self, path: str):
        with open(path, "wb") as f:
            f.write(self.to_bytes())

    @classmethod
    def from_bytes(cls, blob: bytes, tiers: TierTable, meter: TrafficMeter | None = None,
                   *, append_tokens: int = 256) -> "PagedStore":
        """Load an SPHKV1 snapshot into device pages (store.py:391-427).

        The host parses the headers and the pointer table; the page bytes go
        to the device in one copy and `sphkv_import_streams` rebuilds the
        word-interleaved code blocks, swizzled values and protect flags.
        As in the reference, token ids come back as -1 and values as fp16."""
        import torch

        mv = memoryview(blob)
        if bytes(mv[: len(FILE_MAGIC)]) != FILE_MAGIC:
            raise ValueError("bad magic: not a store snapshot")
        off = len(FILE_MAGIC)
        layers, heads, d, d_v, page_size, n_pages = struct.unpack_from("<6I", mv, off)
        off += 24
        hdr, spans = [], []
        for _ in range(n_pages):
            tid, layer, head, _, count, scale = struct.unpack_from("<BBBBId", mv, off)
            off += 16
            t = tiers.spec_for(tid)
            prot_n, tag_n = (count + 7) // 8, (count * t.meta_bits + 7) // 8
            a_n, r_n = packed_nbytes(count * (d - 1), t.angle_bits), packed_nbytes(count, t.radius_bits)
            prot = np.unpackbits(np.frombuffer(mv, np.uint8, prot_n, off))[:count]
            off += prot_n + tag_n
            spans.append((off, a_n + r_n + 2 * count * d_v, prot))
            off += a_n + r_n + 2 * count * d_v
            hdr.append((t, layer, head, count, scale))
        groups = layers * heads
        ptrs = []
        for _ in range(groups):
            (n,) = struct.unpack_from("<Q", mv, off)
            off += 8
            ptrs.append(np.frombuffer(mv, np.uint64, n, off).astype(np.int64))
            off += 8 * n
        per_group = max([len(x) for x in ptrs] + [1])
        store = cls(tiers, layers, heads, d, d_v, page_size, meter,
                    capacity_tokens=per_group * page_size, append_tokens=append_tokens)
        if n_pages + groups > store.max_pages:
            store._grow(n_pages + groups * (len(tiers.non_drop) + 2))
        # page table (file order = page ids), code blocks packed back to back
        rows = np.zeros(n_pages, dtype=_lib.PAGE_DTYPE)
        code_off = 0
        for i, (t, layer, head, count, scale) in enumerate(hdr):
            if layer >= layers or head >= heads or count > page_size:
                raise ValueError(f"page {i}: header outside the store geometry")
            rows[i] = (code_off, scale, np.float32(scale / float((1 << t.radius_bits) - 1)), count,
                       layer * heads + head, t.id, t.angle_bits, t.radius_bits, t.meta_bits)
            code_off += code_block_bytes(d, page_size, t.angle_bits, t.radius_bits)
        if code_off > store.code_cap:
            raise RuntimeError("store pool exhausted")
        ids = [t.id for t in tiers.tiers]
        ptr = np.zeros((groups, store.ptr_cap), dtype=np.int32)
        plen = np.zeros(groups, dtype=np.int32)
        last = np.full((groups, _lib.MAX_TIERS), -1, dtype=np.int32)
        for g, lst in enumerate(ptrs):
            if np.any(lst >= n_pages):
                raise ValueError("pointer table references a missing page")
            ptr[g, : len(lst)] = lst
            plen[g] = len(lst)
            for idx in lst:  # store.py:423-426
                last[g, ids.index(int(rows[idx]["tier"]))] = idx
        # stream blob in the export layout: angle | radius | values | protect bytes
        offs = np.zeros(n_pages + 1, dtype=np.int64)
        for i, (_, ln, prot) in enumerate(spans):
            offs[i + 1] = offs[i] + ln + len(prot)
        buf = np.zeros(int(offs[-1]) + 16, dtype=np.uint8)
        for i, (o, ln, prot) in enumerate(spans):
            buf[offs[i]: offs[i] + ln] = np.frombuffer(mv, np.uint8, ln, o)
            buf[offs[i] + ln: offs[i + 1]] = prot
        dev = "cuda"
        store.t_pages[: n_pages * 32] = torch.as_tensor(rows.view(np.uint8), device=dev)
        store.t_ptr.view(groups, store.ptr_cap).copy_(torch.as_tensor(ptr, device=dev))
        store.t_ptr_len.copy_(torch.as_tensor(plen, device=dev))
        store.t_group_last.copy_(torch.as_tensor(last.reshape(-1), device=dev))
        store.t_counters[0] = n_pages
        store.t_counters[1] = code_off
        l = _lib.require_gpu()
        blob_d = torch.as_tensor(buf, device=dev)
        offs_d = torch.as_tensor(offs[:-1], device=dev)
        _lib.check(l.sphkv_import_streams(store.cptr, n_pages, offs_d.data_ptr(),
                                          blob_d.data_ptr(), _lib.stream_ptr()))
        store._invalidate()
        store._refresh_lut()
        return store

    @classmethod
    def from_file(cls, path: str, tiers: TierTable) -> "PagedStore":
        with open(path, "rb") as f:
            return cls.from_bytes(f.read(), tiers)


def pack_pages_arrays(assignment, radii, angles, values, tiers: TierTable, page_size: int,
                      meter: TrafficMeter | None = None, *, append_tokens: int = 256) -> PagedStore:
    """Pack retained states into a fresh device store (store.py:430-482).

    Inputs are numpy arrays as in the reference: assignment (z, tier,
    protected) over (L, H, T), radii (L, H, T), angles (L, H, T, d-1),
    values (L, H, T, d_v).  Values are stored fp16 (the SPHKV1 value type)."""
    import torch

    radii = np.asarray(radii, dtype=np.float64)
    angles = np.asarray(angles, dtype=np.float64)
    values = np.asarray(values)
    if radii.shape != assignment.z.shape or angles.shape[:3] != radii.shape:
        raise KeyError("assignment references states missing from the key arrays")
    if values.shape[:3] != radii.shape:
        raise KeyError("assignment references states missing from the value arrays")
    if np.any((assignment.z == 1) & (assignment.tier == DROP_TIER_ID)):
        raise ValueError("retained state assigned to the drop tier")
    L, H, T = radii.shape
    d = angles.shape[-1] + 1
    d_v = values.shape[-1]
    store = PagedStore(tiers, L, H, d, d_v, page_size, meter, capacity_tokens=T,
                       append_tokens=append_tokens)
    pack_device(store, radii=radii.reshape(-1), angles=angles.reshape(-1, d - 1),
                values=values.reshape(-1, d_v), z=assignment.z.reshape(-1),
                tier=assignment.tier.reshape(-1), protect=assignment.protected.reshape(-1),
                tokens=T)
    # write meter: headers + pointer entries, code streams, value blocks
    for p in store.pages:
        store.meter.add_write("header", PAGE_HEADER_BYTES + PTR_ENTRY_BYTES)
        store.meter.add_write("k_codes", p.angle_stream_bytes(d) + p.radius_stream_bytes())
        store.meter.add_write("values", p.value_block_bytes(d_v))
    return store


def pack_device(store: PagedStore, *, radii, values, z, tier, protect, tokens, angles=None,
                keys=None, groups=None):
    """Device packer entry (tensors or arrays): encode + quantize + page layout.

    `groups` = (first, count) packs only that contiguous group range (arrays
    relative to it, e.g. one sequence of a batched store); default: all."""
    import torch

    l = _lib.require_gpu()

    def dev(x, dt):
        if x is None:
            return None
        if isinstance(x, torch.Tensor):
            return x.to(device="cuda", dtype=dt).contiguous()
        return torch.as_tensor(np.ascontiguousarray(x), device="cuda").to(dt)

    kd = 0
    k = None
    if keys is not None:
        k = keys if isinstance(keys, torch.Tensor) else dev(keys, torch.float64)
        k = k.contiguous()
        kd = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
              torch.float16: _lib.F16}[k.dtype]
    r = dev(radii, torch.float64)
    a = dev(angles, torch.float64)
    v = _lib.to_f16(values)
    zz = dev(z, torch.int8)
    tt = dev(tier, torch.int16)
    pp = dev(protect, torch.uint8)
    g0, ng = (0, store.groups) if groups is None else (int(groups[0]), int(groups[1]))
    nbytes = (l.sphkv_pack_workspace_bytes(store.batch, store.layers, store.heads, tokens)
              - (store.groups - ng) * tokens * 4)
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    _lib.check(l.sphkv_pack_pages_groups(store.cptr, g0, ng, _lib.ptr(k), kd, _lib.ptr(a),
                                         r.data_ptr(), v.data_ptr(), zz.data_ptr(),
                                         tt.data_ptr(), pp.data_ptr(), tokens, ws.data_ptr(),
                                         nbytes, _lib.stream_ptr()))
    store._invalidate()
    store._refresh_lut()
    return store


class DenseStore:
    """Dense baseline store on the device (store.py:485-569): bf16 keys and
    fp16 values in pages of `page_size`, read by the dense decode kernel."""

    def __init__(self, layers, heads, d, d_v, page_size, meter=None, *, batch=1):
        self.batch, self.layers, self.heads = batch, layers, heads
        self.d, self.d_v, self.page_size = d, d_v, page_size
        self.meter = meter if meter is not None else TrafficMeter()
        self.tokens = 0
        self.t_keys = None
        self.t_values = None
        self.cstruct = None

    def bulk_load(self, keys, values, metered=False, groups=None):
        """keys (B*L*H, T, d) / (L, H, T, d); values likewise with d_v.
        `groups` = (first, count): load only that contiguous group range (the
        arrays then hold those groups only); the pools are sized on first use."""
        import torch

        l = _lib.require_gpu()
        k = keys if isinstance(keys, torch.Tensor) else torch.as_tensor(np.asarray(keys), device="cuda")
        v = values if isinstance(values, torch.Tensor) else torch.as_tensor(np.asarray(values), device="cuda")
        k = k.to("cuda").contiguous()
        v = _lib.to_f16(v)
        all_groups = self.batch * self.layers * self.heads
        g0, ng = (0, all_groups) if groups is None else (int(groups[0]), int(groups[1]))
        T = k.numel() // (ng * self.d)
        P = self.page_size
        npg = -(-T // P)
        if self.cstruct is None:
            self.tokens = T
            dp = (self.d + 15) // 16 * 16
            dvp = (self.d_v + 15) // 16 * 16
            self.t_keys = torch.zeros(all_groups * npg * P * dp, dtype=torch.bfloat16, device="cuda")
            self.t_values = torch.zeros(all_groups * npg * P * dvp, dtype=torch.float16,
                                        device="cuda")
            c = _lib.CDenseStore()
            c.batch, c.layers, c.heads = self.batch, self.layers, self.heads
            c.d, c.d_v, c.page_size = self.d, self.d_v, P
            c.n_pages_per_group, c.tokens = npg, T
            c.keys, c.values = self.t_keys.data_ptr(), self.t_values.data_ptr()
            self.cstruct = c
        elif T != self.tokens:
            raise ValueError(f"dense store holds {self.tokens} tokens per group, got {T}")
        c = self.cstruct
        groups = ng
        kd = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
              torch.float16: _lib.F16}[k.dtype]
        _lib.check(l.sphkv_dense_fill_groups(ctypes.byref(c), g0, ng, k.data_ptr(), kd,
                                             v.data_ptr(), _lib.stream_ptr()))
        if metered:
            for _ in range(groups):
                pages = npg
                self.meter.add_write("header", (PAGE_HEADER_BYTES + PTR_ENTRY_BYTES) * pages)
                self.meter.add_write("dense_k_write", T * self.d * VALUE_BYTES_PER_ENTRY)
                self.meter.add_write("values", T * self.d_v * VALUE_BYTES_PER_ENTRY)

    @property
    def cptr(self):
        return ctypes.byref(self.cstruct)

    def meter_dense_stream(self):
        """Metered dense pass of one (layer, head) (store.py:533-546)."""
        n = self.tokens
        pages = (n + self.page_size - 1) // self.page_size
        self.meter.add_read("header", PAGE_HEADER_BYTES * pages)
        self.meter.add_read("dense_k_read", n * self.d * VALUE_BYTES_PER_ENTRY)
        self.meter.add_read("values", n * self.d_v * VALUE_BYTES_PER_ENTRY)

    def logits(self, group, q):
        """fp32 logits [tokens, G] of one group for q [G, d] (sphkv_dense_store_logits)."""
        import torch

        l = _lib.require_gpu()
        q = q.to(device="cuda", dtype=torch.float32).reshape(-1, self.d).contiguous()
        out = torch.empty((self.tokens, q.shape[0]), dtype=torch.float32, device="cuda")
        _lib.check(l.sphkv_dense_store_logits(self.cptr, q.data_ptr(), q.shape[0], int(group),
                                              out.data_ptr(), _lib.stream_ptr()))
        return out

    def view(self, layer, head, seq=0):
        """Host (keys, values) of one group in token order, un-swizzled from the
        pages (bf16 keys and fp16 values as stored, returned as float64)."""
        import torch

        g = (seq * self.layers + layer) * self.heads + head
        P, T = self.page_size, self.tokens
        dp, dvp = (self.d + 15) // 16 * 16, (self.d_v + 15) // 16 * 16
        npg = self.n_pages_per_group

        def unswz(pool, w, width):
            blk = pool.view(-1, npg * P, w)[g].view(npg, P, w // 8, 8)
            i = torch.arange(P, device=blk.device)
            mask = min(w // 8, 8) - 1
            chunk = torch.arange(w // 8, device=blk.device)[None, :] ^ (i[:, None] & mask)
            rows = torch.gather(blk, 2, chunk[None, :, :, None].expand(npg, P, w // 8, 8))
            return rows.reshape(npg * P, w)[:T, :width].double().cpu().numpy()

        return unswz(self.t_keys, dp, self.d), unswz(self.t_values, dvp, self.d_v)

    def stream_dense(self, layer, head, metered=True):
        """Metered dense view (store.py:533-546): headers + dense K + values."""
        keys, values = self.view(layer, head)
        if metered:
            self.meter_dense_stream()
        return keys, values

    @property
    def n_pages_per_group(self):
        return -(-self.tokens // self.page_size)

    def retained_count(self, layer=None, head=None):
        n = 0
        for l in range(self.layers):
            for h in range(self.heads):
                if (layer is None or l == layer) and (head is None or h == head):
                    n += self.tokens * self.batch
        return n

    def stream_bytes_total(self):
        groups = self.batch * self.layers * self.heads
        return groups * (PAGE_HEADER_BYTES * self.n_pages_per_group
                         + self.tokens * (self.d + self.d_v) * VALUE_BYTES_PER_ENTRY)

    def resident_breakdown(self) -> ResidentBreakdown:
        groups = self.batch * self.layers * self.heads
        br = ResidentBreakdown()
        slot = (self.d + self.d_v) * VALUE_BYTES_PER_ENTRY
        pages = self.n_pages_per_group
        br.payload_bytes = groups * self.tokens * slot
        br.frag_bytes = groups * (pages * self.page_size - self.tokens) * slot
        br.header_bytes = PAGE_HEADER_BYTES * pages * groups
        br.ptr_bytes = FILE_DIRECTORY_BYTES + PTR_ENTRY_BYTES * (groups + pages * groups)
        return br

    def b_kv(self, t_active):
        if t_active < 1:
            raise ValueError("T_active must be >= 1")
        return self.resident_breakdown().total / t_active


def dense_mem_estimate(batch, layers, tokens, heads, d_k, d_v, bytes_per_entry):
    for name, v in (("batch", batch), ("layers", layers), ("tokens", tokens), ("heads", heads),
                    ("d_k", d_k), ("d_v", d_v), ("bytes_per_entry", bytes_per_entry)):
        if v <= 0:
            raise ValueError(f"{name} must be positive")
    return batch * layers * tokens * heads * (d_k + d_v) * bytes_per_entry
