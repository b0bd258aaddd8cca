"""CPU oracle for the Spherical-KV decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (the read-only
`sphkv` package of arXiv 2605.18856, pkg/src/sphkv/*.py).  It exists to check
the B200 CUDA path; it is never the thing measured or shipped.  Only
`tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
reference` legs of `bench.py` may import it.  The product package
(`paper_2605_18856_b200`) must not import it, and does not.

Parity pinning: every function below is checked against golden vectors that
were produced by running the *real* reference in the build container
(`tests/golden/make_golden.py` imports /root/reference/pkg/src and writes
`tests/golden/*.npz`; `tests/test_oracle_golden.py` replays them).

Conventions restated from the reference (file:line into pkg/src/sphkv/):
  * angles: right-to-left tail norms by a *sequential* cumsum, arctan2 chain,
    circular last angle wrapped into [0, 2pi), polar clip  (codec.py:239-257)
  * radius: the batched path's pairwise norm  np.linalg.norm(k, axis=1)
    (decode.py:457).  The 1-D `to_spherical` uses BLAS ddot (codec.py:231);
    the two differ in the last bit for ~18% of keys, so both the oracle and
    the GPU use the pairwise form and feed identical radii everywhere.
  * quantizers by division by the step constants, rint, clip / mod
    (codec.py:318-355), prefill radius code (store.py:465-471)
  * LSB-first bit streams (bitpack.py:14-48), SoA coordinate-major page
    streams with stride = count (store.py:205-211)
  * page order: (layer, head) -> tier ascending -> chunks of <= P in token
    order (store.py:453-480)
  * RDR scoring in numpy's exact fp64 operation order (controller.py:213-245)
  * greedy allocation: lexsort(-nu, l, h, tok) + sequential fit
    (controller.py:301-346); downtier_before_drop (controller.py:349-386)
  * ADA attend: logit = (r_q/sqrt d) * r~ * (feat . qfeat), stable softmax,
    value mix, pointer order (decode.py:123-192, 291-355)
  * SPHKV1 snapshot bytes (store.py:362-388)
"""

from __future__ import annotations

import math
import struct

import numpy as np

TWO_PI = 2.0 * math.pi
NORM_EPS = 1e-12          # codec.py:218
NU_EPS = 1e-12            # controller.py:35
PAGE_HEADER_BYTES = 16    # store.py:38
PTR_ENTRY_BYTES = 8       # store.py:39
VALUE_BYTES = 2           # store.py:40
FILE_MAGIC = b"SPHKV1"    # store.py:41
FILE_DIRECTORY_BYTES = 6 + 24
APPEND_SCALE_HEADROOM = 1.25  # store.py:48


# ---------------------------------------------------------------------------
# tiers / rate model  (codec.py:73-107)
# ---------------------------------------------------------------------------

def rate_bits(tier, d):
    """tier = (id, angle_bits, radius_bits, meta_bits); drop (id 0) costs 0."""
    tid, ba, br, bm = tier
    if tid == 0:
        return 0
    return (d - 1) * ba + br + bm


# ---------------------------------------------------------------------------
# encode  (codec.py:222-257)
# ---------------------------------------------------------------------------

def pairwise_norm(k):
    """Row norms exactly as np.linalg.norm(k, axis=1) (numpy pairwise add)."""
    k = np.asarray(k, dtype=np.float64)
    return np.sqrt(np.add.reduce(k * k, axis=1))


def angles_from_unit(u):
    u = np.asarray(u, dtype=np.float64)
    n, d = u.shape
    out = np.empty((n, d - 1))
    # tail[:, j] = || u[:, j:] ||, accumulated from the right, sequentially
    rev = np.cumsum((u * u)[:, ::-1], axis=1)
    tail = np.sqrt(rev[:, ::-1])
    # column by column, the same strided ufunc calls the reference makes, so
    # numpy's SIMD dispatch (and hence the last ulp) matches it on any host
    for j in range(d - 2):
        out[:, j] = np.arctan2(tail[:, j + 1], u[:, j])
    if d > 2:
        np.clip(out[:, : d - 2], 0.0, math.pi, out=out[:, : d - 2])
    last = np.arctan2(u[:, d - 1], u[:, d - 2])
    out[:, d - 2] = np.where(last < 0, last + TWO_PI, last)
    return out


def encode_batch(keys):
    """Dense rows (n, d) -> (radii (n,), angles (n, d-1)); zero rows -> 0 angles."""
    keys = np.asarray(keys, dtype=np.float64)
    r = pairwise_norm(keys)
    ang = angles_from_unit(keys / (r[:, None] + NORM_EPS))
    ang[r == 0.0] = 0.0
    return r, ang


# ---------------------------------------------------------------------------
# quantizers  (codec.py:318-389, store.py:465-471)
# ---------------------------------------------------------------------------

def polar_step(bits):
    return math.pi / float((1 << bits) - 1)


def circular_step(bits):
    return TWO_PI / float(1 << bits)


def quantize_angles(angles, bits):
    angles = np.asarray(angles, dtype=np.float64)
    dm1 = angles.shape[-1]
    codes = np.empty(angles.shape, dtype=np.uint64)
    top = float((1 << bits) - 1)
    if dm1 > 1:
        codes[..., : dm1 - 1] = np.clip(
            np.rint(angles[..., : dm1 - 1] / polar_step(bits)), 0, top).astype(np.uint64)
    circ = np.rint(angles[..., dm1 - 1] / circular_step(bits)).astype(np.int64)
    codes[..., dm1 - 1] = np.mod(circ, np.int64(1 << bits)).astype(np.uint64)
    return codes


def dequantize_angles(codes, bits):
    codes = np.asarray(codes, dtype=np.uint64)
    dm1 = codes.shape[-1]
    out = np.empty(codes.shape, dtype=np.float64)
    if dm1 > 1:
        out[..., : dm1 - 1] = codes[..., : dm1 - 1].astype(np.float64) * polar_step(bits)
    out[..., dm1 - 1] = codes[..., dm1 - 1].astype(np.float64) * circular_step(bits)
    return out


def prefill_radius_codes(radii, scale, bits):
    levels = float((1 << bits) - 1)
    return np.rint(np.clip(np.asarray(radii, np.float64) / scale, 0.0, 1.0)
                   * levels).astype(np.uint64)


def append_radius_code(r, scale, bits):
    """Python round() (banker's) of the clamped ratio (codec.py:353-355)."""
    levels = (1 << bits) - 1
    return int(round(min(max(r / scale, 0.0), 1.0) * levels))


# ---------------------------------------------------------------------------
# bit streams  (bitpack.py)
# ---------------------------------------------------------------------------

def packed_nbytes(count, bits):
    return (count * bits + 7) // 8


def pack_bits(codes, bits):
    codes = np.asarray(codes, dtype=np.uint64).ravel()
    if codes.size == 0:
        return np.zeros(0, dtype=np.uint8)
    planes = ((codes[:, None] >> np.arange(bits, dtype=np.uint64)[None, :])
              & np.uint64(1)).astype(np.uint8)
    return np.packbits(planes.ravel(), bitorder="little")[: packed_nbytes(codes.size, bits)]


def unpack_bits(stream, bits, count):
    stream = np.asarray(stream, dtype=np.uint8)
    flat = np.unpackbits(stream, bitorder="little")[: count * bits]
    planes = flat.reshape(count, bits).astype(np.uint64)
    return (planes << np.arange(bits, dtype=np.uint64)[None, :]).sum(axis=1).astype(np.uint64)


# ---------------------------------------------------------------------------
# pages  (store.py:136-211, 430-482)
# ---------------------------------------------------------------------------

class OraclePage:
    __slots__ = ("tier", "layer", "head", "count", "scale", "angle_codes",
                 "radius_codes", "values", "protect", "token_ids")

    def __init__(self, tier, layer, head, scale, d, d_v, capacity):
        self.tier = tier  # (id, ba, br, bm)
        self.layer, self.head = layer, head
        self.count = 0
        self.scale = float(scale)
        self.angle_codes = np.zeros((capacity, d - 1), dtype=np.uint64)
        self.radius_codes = np.zeros(capacity, dtype=np.uint64)
        self.values = np.zeros((capacity, d_v), dtype=np.float64)
        self.protect = np.zeros(capacity, dtype=bool)
        self.token_ids = np.full(capacity, -1, dtype=np.int64)

    def angle_stream(self):
        """Coordinate-major SoA stream with stride = count (store.py:205-208)."""
        return pack_bits(self.angle_codes[: self.count].T.reshape(-1), self.tier[1])

    def radius_stream(self):
        return pack_bits(self.radius_codes[: self.count], self.tier[2])


class OracleStore:
    """Page list + pointer table, the state of a reference PagedStore."""

    def __init__(self, tiers, layers, heads, d, d_v, page_size):
        self.tiers = list(tiers)
        self.layers, self.heads, self.d, self.d_v = layers, heads, d, d_v
        self.page_size = page_size
        self.pages = []
        self.pointer = {(l, h): [] for l in range(layers) for h in range(heads)}
        self.group_last = {}

    def tier(self, tid):
        for t in self.tiers:
            if t[0] == tid:
                return t
        raise KeyError(tid)

    def open_page(self, l, h, tier, scale):
        p = OraclePage(tier, l, h, scale, self.d, self.d_v, self.page_size)
        self.pages.append(p)
        idx = len(self.pages) - 1
        self.pointer[(l, h)].append(idx)
        self.group_last[(l, h, tier[0])] = idx
        return p

    # store.py:178-203
    def page_bytes(self, p):
        d, dv = self.d, self.d_v
        ang = packed_nbytes(p.count * (d - 1), p.tier[1])
        rad = packed_nbytes(p.count, p.tier[2])
        val = p.count * dv * VALUE_BYTES
        tag = (p.count * p.tier[3] + 7) // 8
        prot = (p.count + 7) // 8
        slot = ((d - 1) * p.tier[1] + p.tier[2] + p.tier[3] + 7) // 8 + dv * VALUE_BYTES
        frag = (self.page_size - p.count) * slot
        return ang, rad, val, tag, prot, frag

    def expected_stream_bytes(self, l, h):
        total = 0
        for idx in self.pointer[(l, h)]:
            ang, rad, val, *_ = self.page_bytes(self.pages[idx])
            total += PAGE_HEADER_BYTES + ang + rad + val
        return total

    def resident_breakdown(self):
        out = dict(payload=0, header=0, ptr=0, tag=0, prot=0, frag=0)
        for p in self.pages:
            ang, rad, val, tag, prot, frag = self.page_bytes(p)
            out["payload"] += ang + rad + val
            out["tag"] += tag
            out["prot"] += prot
            out["frag"] += frag
        out["header"] = PAGE_HEADER_BYTES * len(self.pages)
        out["ptr"] = FILE_DIRECTORY_BYTES + PTR_ENTRY_BYTES * (
            self.layers * self.heads + len(self.pages))
        out["total"] = sum(out[k] for k in ("payload", "header", "ptr", "tag", "prot", "frag"))
        return out

    def to_bytes(self):
        """SPHKV1 snapshot (store.py:362-388)."""
        parts = [FILE_MAGIC, struct.pack("<6I", self.layers, self.heads, self.d,
                                         self.d_v, self.page_size, len(self.pages))]
        for p in self.pages:
            parts.append(struct.pack("<BBBBId", p.tier[0], p.layer, p.head, 0,
                                     p.count, p.scale))
            parts.append(np.packbits(p.protect[: p.count]).tobytes())  # MSB-first
            parts.append(b"\x00" * ((p.count * p.tier[3] + 7) // 8))
            parts.append(p.angle_stream().tobytes())
            parts.append(p.radius_stream().tobytes())
            parts.append(p.values[: p.count].astype(np.float16).tobytes())
        for l in range(self.layers):
            for h in range(self.heads):
                idxs = self.pointer[(l, h)]
                parts.append(struct.pack("<Q", len(idxs)))
                parts.append(np.asarray(idxs, dtype=np.uint64).tobytes())
        return b"".join(parts)

    # store.py:249-274 (append path) + codec.py:365-377
    def append_item(self, l, h, radius, angles, value, tier_id, protected=False,
                    token_id=-1):
        if tier_id == 0:
            return None
        tier = self.tier(tier_id)
        idx = self.group_last.get((l, h, tier_id))
        page = self.pages[idx] if idx is not None else None
        if page is None or page.count >= self.page_size or radius > page.scale:
            scale = max(radius * APPEND_SCALE_HEADROOM, 1e-9)
            if page is None and radius == 0.0:
                scale = 1e-9
            page = self.open_page(l, h, tier, scale)
        if radius > page.scale * (1 + 1e-12):
            raise ValueError("radius exceeds page scale")
        i = page.count
        page.angle_codes[i] = quantize_angles(np.asarray(angles)[None, :], tier[1])[0]
        page.radius_codes[i] = append_radius_code(radius, page.scale, tier[2])
        page.values[i] = value
        page.protect[i] = protected
        page.token_ids[i] = token_id
        page.count += 1
        return page


def pack_pages(tiers, z, tier_of, protected, radii, angles, values, page_size):
    """pack_pages_arrays restated (store.py:430-482).

    z, tier_of, protected: (L, H, T); radii (L, H, T); angles (L, H, T, d-1);
    values (L, H, T, d_v).  Returns an OracleStore."""
    L, H, T = radii.shape
    d = angles.shape[-1] + 1
    d_v = values.shape[-1]
    if np.any((z == 1) & (tier_of == 0)):
        raise ValueError("retained state assigned to the drop tier")
    st = OracleStore(tiers, L, H, d, d_v, page_size)
    for l in range(L):
        for h in range(H):
            for t in tiers[1:]:
                toks = np.flatnonzero((z[l, h] == 1) & (tier_of[l, h] == t[0]))
                for s in range(0, toks.size, page_size):
                    ch = toks[s: s + page_size]
                    scale = max(float(radii[l, h, ch].max()), 1e-9)
                    p = st.open_page(l, h, t, scale)
                    n = ch.size
                    p.angle_codes[:n] = quantize_angles(angles[l, h, ch], t[1])
                    p.radius_codes[:n] = prefill_radius_codes(radii[l, h, ch], scale, t[2])
                    p.values[:n] = values[l, h, ch]
                    p.protect[:n] = protected[l, h, ch]
                    p.token_ids[:n] = ch
                    p.count = n
    return st


# ---------------------------------------------------------------------------
# RDR  (controller.py:163-386)
# ---------------------------------------------------------------------------

def score_states(radii, u_hat, s_hat, r_q, omega, segments, alpha_theta, alpha_r,
                 tiers, eps, lam, protected, d):
    """Vectorized scoring in numpy's fp64 operation order (controller.py:219-245).

    tiers: list of (id, ba, br, bm), drop first; eps: {id: (eps_theta, eps_r)}.
    Returns dict(best_tier, score, nu, d_drop, w_theta, w_r)."""
    L, H, T = radii.shape
    sqrt_d = math.sqrt(d)
    om = np.asarray(omega, dtype=np.float64)[np.asarray(segments)].astype(np.float64)[None, None, :]
    w_theta = alpha_theta * np.asarray(u_hat)[:, :, None] * om * (r_q * radii / sqrt_d)
    w_r = alpha_r * (1.0 - np.asarray(s_hat)[:, :, None]) * om * (r_q / sqrt_d)
    d_drop = w_theta + w_r
    best = np.zeros((L, H, T), dtype=np.int16)
    score = -d_drop.copy()
    score[protected] = -np.inf
    for t in tiers[1:]:
        et, er = eps[t[0]]
        s = -(w_theta * et + w_r * er) - lam * rate_bits(t, d)
        upd = s > score
        score = np.where(upd, s, score)
        best = np.where(upd, np.int16(t[0]), best)
    d_best = np.empty_like(d_drop)
    r_best = np.empty_like(d_drop)
    for t in tiers:
        m = best == t[0]
        if not m.any():
            continue
        et, er = (1.0, 1.0) if t[0] == 0 else eps[t[0]]
        d_best[m] = (w_theta * et + w_r * er)[m]
        r_best[m] = rate_bits(t, d)
    nu = (d_drop - d_best) / (r_best + NU_EPS)
    return dict(best_tier=best, score=score, nu=nu, d_drop=d_drop,
                w_theta=w_theta, w_r=w_r)


def score_one(radius, u_hat_lh, s_hat_lh, r_q, om, alpha_theta, alpha_r, tiers, eps,
              lam, d, protected=False):
    """score_and_best_tier restated with Python scalars (controller.py:163-198)."""
    sqrt_d = math.sqrt(d)
    w_theta = alpha_theta * u_hat_lh * om * (r_q * radius / sqrt_d)
    w_r = alpha_r * (1.0 - s_hat_lh) * om * (r_q / sqrt_d)

    def dist(tid):
        et, er = (1.0, 1.0) if tid == 0 else eps[tid]
        return w_theta * et + w_r * er

    best_id, best_s = None, -math.inf
    for t in (tiers[1:] if protected else tiers):
        s = -dist(t[0]) - lam * rate_bits(t, d)
        if s > best_s:
            best_id, best_s = t[0], s
    rate = rate_bits([t for t in tiers if t[0] == best_id][0], d)
    nu = (dist(0) - dist(best_id)) / (rate + NU_EPS)
    return best_id, best_s, nu


class Infeasible(Exception):
    pass


def allocate_greedy(best_tier, nu, protected, budget_bits, tiers, d):
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    L, H, T = best_tier.shape
    z = np.zeros((L, H, T), dtype=np.int8)
    tier = np.zeros((L, H, T), dtype=np.int16)
    max_t = tiers[-1]
    n_prot = int(np.count_nonzero(protected))
    remaining = budget_bits - n_prot * rate_bits(max_t, d)
    if remaining < 0:
        raise Infeasible("protected demand exceeds budget")
    z[protected] = 1
    tier[protected] = max_t[0]
    rate = {t[0]: rate_bits(t, d) for t in tiers}
    flat_free = np.flatnonzero(~protected.ravel())
    keys = -nu.ravel()[flat_free]
    order = flat_free[np.argsort(keys, kind="stable")]  # ties: flat (l, h, tok) order
    bt = best_tier.ravel()
    zf, tf = z.ravel(), tier.ravel()
    for f in order:
        t = int(bt[f])
        if t == 0:
            continue
        c = rate[t]
        if c <= remaining:
            zf[f] = 1
            tf[f] = t
            remaining -= c
    return z, tier


def full_best_tier(best_tier, protected, tiers):
    tier = best_tier.copy()
    tier[protected] = tiers[-1][0]
    return (tier != 0).astype(np.int8), tier


def downtier_before_drop(z0, tier0, nu, protected, budget_bits, tiers, d):
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    z, tier = z0.copy(), tier0.copy()
    rate = {t[0]: rate_bits(t, d) for t in tiers}
    ids = [t[0] for t in tiers]
    below = {ids[k]: ids[k - 1] for k in range(1, len(ids))}
    total = sum(rate[int(t)] for t in tier.ravel())
    if total <= budget_bits:
        return z, tier
    flat_free = np.flatnonzero(~protected.ravel())
    order = flat_free[np.argsort(nu.ravel()[flat_free], kind="stable")]
    zf, tf = z.ravel(), tier.ravel()
    for f in order:
        while total > budget_bits and tf[f] != 0:
            cur = int(tf[f])
            nxt = below[cur]
            total -= rate[cur] - rate[nxt]
            tf[f] = nxt
            if nxt == 0:
                zf[f] = 0
        if total <= budget_bits:
            break
    if total > budget_bits:
        raise Infeasible("protected demand exceeds budget")
    return z, tier


# ---------------------------------------------------------------------------
# attend  (decode.py:63-87, 123-192, 291-355)
# ---------------------------------------------------------------------------

def angular_features(angles):
    angles = np.atleast_2d(np.asarray(angles, dtype=np.float64))
    n, dm1 = angles.shape
    c, s = np.cos(angles), np.sin(angles)
    prods = np.cumprod(s, axis=1)
    out = np.empty((n, dm1 + 1))
    out[:, 0] = c[:, 0]
    out[:, 1:dm1] = prods[:, : dm1 - 1] * c[:, 1:]
    out[:, dm1] = prods[:, dm1 - 1]
    return out


def query_features(q):
    """(r_q, qfeat) as the rollout's batched query path (decode.py:418-422)."""
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    r = pairwise_norm(q)
    u = q / (r[:, None] + NORM_EPS)
    return r, angular_features(angles_from_unit(u))


class FeatureCache:
    """Per-page decoded radii and feature rows (decode.py:123-160 memoization)."""

    def __init__(self):
        self.cache = {}

    def get(self, store, idx):
        p = store.pages[idx]
        hit = self.cache.get(idx)
        if hit is not None and hit[0] == p.count:
            return hit[1], hit[2]
        ang = dequantize_angles(p.angle_codes[: p.count], p.tier[1])
        feat = angular_features(ang) if p.count else np.zeros((0, store.d))
        levels = float((1 << p.tier[2]) - 1)
        radii = p.radius_codes[: p.count].astype(np.float64) / levels * p.scale
        self.cache[idx] = (p.count, feat, radii)
        return feat, radii


def head_attend(store, l, h, r_q, qfeat, cache=None):
    """Angle-path logits (pointer order), softmax, value mix for one query."""
    cache = cache or FeatureCache()
    scale = math.sqrt(store.d)
    segs, blocks = [], []
    for idx in store.pointer[(l, h)]:
        p = store.pages[idx]
        if p.count == 0:
            continue
        feat, radii = cache.get(store, idx)
        segs.append((r_q / scale) * radii * (feat @ qfeat))
        blocks.append(p.values[: p.count])
    if not segs:
        return np.empty(0), np.zeros(store.d_v)
    logits = np.concatenate(segs)
    w = np.exp(logits - logits.max())
    w /= w.sum()
    out = np.zeros(store.d_v)
    pos = 0
    for b in blocks:
        out += w[pos: pos + b.shape[0]] @ b
        pos += b.shape[0]
    return logits, out


def dense_attend(q, keys, values):
    """Dense reference path (decode.py:63-75, 302-307)."""
    q = np.asarray(q, dtype=np.float64)
    logits = np.asarray(keys, np.float64) @ q / math.sqrt(q.shape[0])
    if logits.size == 0:
        return logits, np.zeros(values.shape[-1])
    w = np.exp(logits - logits.max())
    w /= w.sum()
    return logits, w @ np.asarray(values, np.float64)


def lse_merge(m, lsum, acc):
    """Combine split partials (S, ...) -> output.  Empty splits carry m=-inf,
    l=0, acc=0; all-empty -> zeros (decode.py:345-346)."""
    m = np.asarray(m, np.float64)
    M = m.max(axis=0)
    safe = np.where(np.isfinite(M), M, 0.0)
    wgt = np.where(np.isfinite(m), np.exp(m - safe[None]), 0.0)
    L = (wgt * lsum).sum(axis=0)
    A = (wgt[..., None] * acc).sum(axis=0)
    out = np.where(L[..., None] > 0, A / np.where(L > 0, L, 1.0)[..., None], 0.0)
    return out


# ---------------------------------------------------------------------------
# host-only workload pieces for bench.py's reference arm (no product code):
# one (layer, kv-head) slice generated, calibrated, scored, allocated and
# packed entirely here, in numpy
# ---------------------------------------------------------------------------

PREFIX_FRAC = 2944 / 4096     # pkg/configs/panel.cfg:8
RETRIEVED_FRAC = 3584 / 4096  # pkg/configs/panel.cfg:9


def segments_for(T):
    seg = np.full(T, 2, dtype=np.int8)
    seg[: int(round(T * PREFIX_FRAC))] = 0
    seg[int(round(T * PREFIX_FRAC)): int(round(T * RETRIEVED_FRAC))] = 1
    return seg


def generate_slice(T, d, G, seed, outlier_frac=0.01, outlier_mult=4.0, query_gain=4.0):
    """One (layer, kv-head) slice of the reference workload distribution
    (workload.py:204-248): unit topic; prefix tokens -topic + 0.35 N/sqrt(d),
    radius |N(1.6, 0.15)|; retrieved/recent topic + 0.6 N/sqrt(d), radius
    |N(1.0, 0.2)|; 1% outliers x4; values N(0, 1); G queries topic + 0.5
    N/sqrt(d) with norm 4 sqrt(d) |N(1, 0.05)|.  Keys are rounded to bf16 and
    values to fp16 as the benchmark stores them.  Returns (keys, values, q,
    prefill-row queries for the features, segments)."""
    rng = np.random.default_rng(seed)
    topic = rng.standard_normal(d)
    topic /= np.linalg.norm(topic)
    seg = segments_for(T)
    pre = (seg == 0)[:, None]
    g = rng.standard_normal((T, d)) / np.sqrt(d)
    base = np.where(pre, -topic + 0.35 * g, topic + 0.6 * g)
    base /= np.linalg.norm(base, axis=-1, keepdims=True)
    radii = np.where(pre[:, 0], np.abs(rng.normal(1.6, 0.15, T)), np.abs(rng.normal(1.0, 0.2, T)))
    radii = np.where(rng.random(T) < outlier_frac, radii * outlier_mult, radii)
    keys = _bf16(base * radii[:, None])
    values = rng.standard_normal((T, d)).astype(np.float16).astype(np.float64)

    def qdraw(n):
        qd = topic + 0.5 * rng.standard_normal((n, d)) / np.sqrt(d)
        qd /= np.linalg.norm(qd, axis=-1, keepdims=True)
        return qd * (query_gain * np.sqrt(d) * np.abs(rng.normal(1.0, 0.05, (n, 1))))

    q = qdraw(G).astype(np.float32).astype(np.float64)
    return keys, values, q, qdraw, seg


def _bf16(x):
    """Round fp64 -> bf16 (nearest-even via fp32) -> fp64, as the benchmark stores keys."""
    f = np.asarray(x, dtype=np.float32)
    b = f.view(np.uint32).astype(np.uint64)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16) << 16
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def features_slice(keys, qdraw, rows=512, seed=1):
    """controller.compute_features (controller.py:99-142) for one slice: a
    causal softmax over <= `rows` sampled prefill rows.  With a single head the
    per-(l, h) normalization gives u_hat = 1 and s_hat = 0 (stated in the
    reference arm's sample description).  Returns (u_raw, inv_margin, r_q)."""
    T, d = keys.shape
    window = max(T // 8, 1)
    idx = np.unique(np.round(np.linspace(0, T - 1, min(rows, T))).astype(int))
    q = qdraw(len(idx))
    logits = q @ keys.T / math.sqrt(d)
    mask = np.arange(T)[None, :] > idx[:, None]
    logits = np.where(mask, -np.inf, logits)
    z = logits - logits.max(axis=1, keepdims=True)
    w = np.exp(z)
    w /= w.sum(axis=1, keepdims=True)
    old = np.arange(T)[None, :] <= (idx[:, None] - window)
    u_raw = float(np.mean(np.sum(np.where(old, w, 0.0), axis=1)))
    ok = idx >= 1
    top2 = np.partition(logits[ok], -2, axis=1)[:, -2:]
    inv_m = float(np.mean(1.0 / (top2[:, 1] - top2[:, 0] + 1e-6)))
    return u_raw, inv_m, float(np.mean(np.linalg.norm(q, axis=-1)))


def calibrate(tiers, sample_keys, seed):
    """TierTable.calibrate / calibrate_distortion (codec.py:172-176, 485-522):
    eps_theta = RMS difference of the angular recurrence on exact vs coded
    key angles against seeded random query directions; eps_r = RMS radius
    decode error over the sample's max-radius scale.  Returns {id: (eps_t, eps_r)}."""
    r, k_ang = encode_batch(np.asarray(sample_keys, dtype=np.float64))
    out = {}
    for t in tiers:
        if t[0] == 0:
            continue
        rng = np.random.default_rng(seed)
        n, d = k_ang.shape[0], k_ang.shape[1] + 1
        k_dec = dequantize_angles(quantize_angles(k_ang, t[1]), t[1])
        q = rng.standard_normal((n, d))
        q /= np.linalg.norm(q, axis=1, keepdims=True) + NORM_EPS
        qa = angles_from_unit(q)

        def paired(qa_, ka):
            cq, sq = np.cos(qa_), np.sin(qa_)
            ck, sk = np.cos(ka), np.sin(ka)
            prods = np.cumprod(sq * sk, axis=1)
            acc = cq[:, 0] * ck[:, 0]
            acc = acc + np.sum(prods[:, :-1] * cq[:, 1:] * ck[:, 1:], axis=1)
            return acc + prods[:, -1]

        eps_t = math.sqrt(float(np.sum((paired(qa, k_ang) - paired(qa, k_dec)) ** 2)) / n)
        scale = float(r.max()) + NORM_EPS
        levels = float((1 << t[2]) - 1)
        codes = np.array([int(round(min(max(x / scale, 0.0), 1.0) * levels)) for x in r])
        eps_r = math.sqrt(float(np.mean(((codes / levels * scale - r) / scale) ** 2)))
        out[t[0]] = (eps_t, eps_r)
    return out


def resident_total(z, tier, tiers, d, d_v, P):
    """Resident bytes (store.py:178-203, 326-336) of one (l, h) slice's pages."""
    total, n_pages = 0, 0
    for t in tiers:
        if t[0] == 0:
            continue
        c = int(np.count_nonzero((z == 1) & (tier == t[0])))
        full, rem = c // P, c % P

        def page_bytes(n):
            return (packed_nbytes(n * (d - 1), t[1]) + packed_nbytes(n, t[2]) + n * d_v * 2
                    + (n * t[3] + 7) // 8 + (n + 7) // 8)

        slot = ((d - 1) * t[1] + t[2] + t[3] + 7) // 8 + d_v * 2
        total += full * page_bytes(P) + (page_bytes(rem) + (P - rem) * slot if rem else 0)
        n_pages += full + (1 if rem else 0)
    return total + PAGE_HEADER_BYTES * n_pages + FILE_DIRECTORY_BYTES + PTR_ENTRY_BYTES * (1 + n_pages)
