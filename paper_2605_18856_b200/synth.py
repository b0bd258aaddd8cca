"""Synthetic KV workloads on the GPU and the prefill pipeline (encode -> RDR -> pack).

The distribution restates the reference generator (workload.py:204-248,
SURVEY.md 8(d)): per-(seq, layer, kv-head) unit topic; prefix tokens point
away from it (radius |N(1.6, 0.15)|), retrieved/recent tokens along it
(radius |N(1.0, 0.2)|), 1% outliers x4, values N(0, 1); each of the G query
heads is topic + 0.5 N/sqrt(d) with norm 4 sqrt(d) |N(1, 0.05)|.  Keys are
stored bf16 and values fp16, as in the benchmark spec.  Generated directly on
the device with a seeded torch.Generator (c2-c5 do not fit on the host).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PREFIX_FRAC = 2944 / 4096     # pkg/configs/panel.cfg:8
RETRIEVED_FRAC = 3584 / 4096  # pkg/configs/panel.cfg:9

PANEL_TIERS = ((0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 6, 8, 8), (4, 7, 8, 8),
               (5, 12, 14, 8), (6, 15, 16, 8))  # pkg/configs/panel.cfg:50-56
PANEL_LAMBDA = 3e-5           # panel.cfg:23
PANEL_OMEGA = (0.02, 2.0, 1.0)  # panel.cfg:24-26


@dataclass
class Workload:
    batch: int
    layers: int
    heads: int
    G: int
    tokens: int
    d: int
    d_v: int
    keys: "object"      # bf16 [B*L*H, T, d]
    values: "object"    # fp16 [B*L*H, T, d_v]
    queries: "object"   # fp32 [B*L*H, G, d]
    topic: "object"     # fp32 [B*L*H, d]
    segments: np.ndarray  # int8 [T]

    @property
    def groups(self):
        return self.batch * self.layers * self.heads


def segments_for(T: int) -> np.ndarray:
    seg = np.full(T, 2, dtype=np.int8)
    seg[: int(round(T * PREFIX_FRAC))] = 0
    seg[int(round(T * PREFIX_FRAC)): int(round(T * RETRIEVED_FRAC))] = 1
    return seg


def generate(batch, layers, heads, G, tokens, d, d_v=None, seed=0, chunk_groups=16,
             outlier_frac=0.01, outlier_mult=4.0, query_gain=4.0):
    import torch

    d_v = d if d_v is None else d_v
    groups = batch * layers * heads
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    seg = segments_for(tokens)
    is_prefix = torch.as_tensor(seg == 0, device="cuda")
    topic = torch.randn((groups, d), generator=gen, device="cuda")
    topic = topic / topic.norm(dim=-1, keepdim=True)
    keys = torch.empty((groups, tokens, d), dtype=torch.bfloat16, device="cuda")
    values = torch.empty((groups, tokens, d_v), dtype=torch.float16, device="cuda")
    sd = 1.0 / math.sqrt(d)
    for g0 in range(0, groups, chunk_groups):
        g1 = min(groups, g0 + chunk_groups)
        n = g1 - g0
        tp = topic[g0:g1, None, :]
        noise = torch.randn((n, tokens, d), generator=gen, device="cuda") * sd
        base = torch.where(is_prefix[None, :, None], -tp + 0.35 * noise, tp + 0.6 * noise)
        base = base / base.norm(dim=-1, keepdim=True)
        r_pre = torch.randn((n, tokens), generator=gen, device="cuda").mul_(0.15).add_(1.6).abs_()
        r_al = torch.randn((n, tokens), generator=gen, device="cuda").mul_(0.2).add_(1.0).abs_()
        radii = torch.where(is_prefix[None, :], r_pre, r_al)
        if outlier_frac > 0:
            out = torch.rand((n, tokens), generator=gen, device="cuda") < outlier_frac
            radii = torch.where(out, radii * outlier_mult, radii)
        keys[g0:g1] = (base * radii[..., None]).to(torch.bfloat16)
        values[g0:g1] = torch.randn((n, tokens, d_v), generator=gen, device="cuda").to(torch.float16)
        del noise, base
    qn = torch.randn((groups, G, d), generator=gen, device="cuda") * sd
    qd = topic[:, None, :] + 0.5 * qn
    qd = qd / qd.norm(dim=-1, keepdim=True)
    qnorm = query_gain * math.sqrt(d) * (torch.randn((groups, G, 1), generator=gen,
                                                     device="cuda") * 0.05 + 1.0).abs()
    queries = (qd * qnorm).float().contiguous()
    return Workload(batch, layers, heads, G, tokens, d, d_v, keys, values, queries, topic, seg)


def features(wl: Workload, rows=512, seed=1):
    """u_hat / s_hat / r_q per (seq, layer, kv-head) from a sampled dense prefill
    pass (controller.py:99-142 recipe, the fp64 sphkv_controller_stats kernel;
    GQA: the G query heads' sampled rows of a KV head are pooled).  The prefill
    queries at the sampled rows are drawn from the workload's query
    distribution.  Returns fp64 numpy (B*L*H,), (B*L*H,), float."""
    import torch
    from .controller import controller_stats_device, feature_rows, normalize_features

    T, d, G = wl.tokens, wl.d, wl.G
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    window = max(T // 8, 1)
    r_idx = feature_rows(T, rows)
    R = len(r_idx)
    u_raw = np.zeros(wl.groups)
    inv_m = np.zeros(wl.groups)
    qnorms = []
    chunk = 64
    for g0 in range(0, wl.groups, chunk):
        g1 = min(wl.groups, g0 + chunk)
        tp = wl.topic[g0:g1].double()
        qn = torch.randn((g1 - g0, G, R, d), generator=gen, device="cuda",
                         dtype=torch.float64) / math.sqrt(d)
        qd = tp[:, None, None, :] + 0.5 * qn
        q = qd / qd.norm(dim=-1, keepdim=True) * (4.0 * math.sqrt(d))
        qnorms.append(q.norm(dim=-1).mean(dim=(1, 2)))
        u, m = controller_stats_device(wl.keys[g0:g1], q.reshape(-1, R, d), r_idx, window)
        u_raw[g0:g1] = u.view(-1, G).mean(-1).cpu().numpy()
        inv_m[g0:g1] = m.view(-1, G).mean(-1).cpu().numpy()
    u_hat, s_hat = normalize_features(u_raw, inv_m)
    r_q = float(torch.cat(qnorms).mean())
    return u_hat, s_hat, r_q


def panel_tiers(eps=None, d=128, sample_keys=None, seed=0):
    """Panel tier table (panel.cfg:50-56), calibrated on a 512-key sample
    (cli.py:72-81 recipe) unless eps constants are given."""
    from .codec import SphericalKey, TierSpec, TierTable, encode_batch

    t = TierTable(tuple(TierSpec(*x) for x in PANEL_TIERS))
    if eps is not None:
        for tid, (a, b) in eps.items():
            t.eps_theta[tid], t.eps_r[tid] = a, b
        return t
    r, a = encode_batch(np.asarray(sample_keys, dtype=np.float64))
    t.calibrate([SphericalKey(float(r[i]), a[i]) for i in range(len(r))], seed)
    return t


def resident_total(counts, tiers, d, d_v, P, groups):
    """Closed-form resident bytes from per-(group, tier) retained counts
    (store.py:178-203, 326-336)."""
    counts = np.asarray(counts, dtype=np.int64)  # [groups, n_tiers]
    total = 0
    n_pages = 0
    for k, t in enumerate(tiers.tiers):
        if t.id == 0:
            continue
        c = counts[:, k]
        pages = -(-c // P)
        n_pages += int(pages.sum())
        ang = (c * (d - 1) * t.angle_bits + 7) // 8
        rad = (c * t.radius_bits + 7) // 8
        val = c * d_v * 2
        # per page formulas summed: pages are full except the last of each group
        full = c // P
        rem = c - full * P
        def page_bytes(n):
            return ((n * (d - 1) * t.angle_bits + 7) // 8 + (n * t.radius_bits + 7) // 8
                    + n * d_v * 2 + (n * t.meta_bits + 7) // 8 + (n + 7) // 8)
        slot = ((d - 1) * t.angle_bits + t.radius_bits + t.meta_bits + 7) // 8 + d_v * 2
        total += int((full * page_bytes(P)).sum() + np.where(rem > 0, page_bytes(rem), 0).sum())
        total += int(np.where(rem > 0, (P - rem) * slot, 0).sum())
        del ang, rad, val
    total += 16 * n_pages + 30 + 8 * (groups + n_pages)
    return total


def dense_resident_total(groups, T, d, d_v, P):
    pages = -(-T // P)
    slot = (d + d_v) * 2
    return groups * (T * slot + (pages * P - T) * slot + 16 * pages) + 30 + 8 * (groups + groups * pages)
