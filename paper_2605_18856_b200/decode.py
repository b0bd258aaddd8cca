"""Decode paths on the B200 (drop-in for sphkv.decode, pkg/src/sphkv/decode.py).

angle  -- `sphkv_ada_decode`: logits straight from radius/angle codes in HBM
          pages (no dense key is ever formed), fp32 online softmax, P.V on the
          tensor cores, split partials merged by `sphkv_lse_merge`.
dense  -- `sphkv_dense_decode`: the bf16 paged baseline with the same
          scheduler, page size and partial/merge contract.
recon  -- the negative control (decode.py:195-217): `sphkv_recon_keys` decodes
          pages into dense key rows (the staging write), the dot re-reads them.

Batched entry points take device tensors: q fp32 [groups, G, d] with the GQA
mapping "a reference head is a KV head; each of its G query heads is an
independent oracle call on the same store".  The reference-
shaped functions (`angle_logits`, `_head_attend`, ...) wrap them for numpy
callers.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .plan import DecodePlan, plan_dense, plan_store

PATHS = ("dense", "angle", "recon")


@dataclass
class AttentionOutput:
    weights: np.ndarray
    output: np.ndarray


def _partials(plan, G, d_v):
    import torch

    floats = G * (d_v + 2)
    return torch.empty((plan.n_slots + 1) * floats, dtype=torch.float32, device="cuda")


def ada_decode(store, q, plan: DecodePlan | None = None, *, out=None, partials=None,
               logits=None, margins=None, stream=None):
    """ADA paged decode over the planned groups.

    q: fp32 device tensor [store.groups, G, d] (rows of unplanned groups are
    ignored).  Returns out [len(plan.group_ids) * G, d_v] fp32 in plan order.
    `logits`, if given, is an fp32 device buffer receiving every logit
    (pointer order per group, G values per item) for parity checks."""
    import torch

    l = _lib.require_gpu()
    if plan is None:
        plan = plan_store(store)
    G = q.shape[-2]
    assert q.dtype == torch.float32 and q.is_contiguous()
    if partials is None:
        partials = _partials(plan, G, store.d_v)
    ng = len(plan.group_ids)
    if out is None:
        out = torch.empty((ng * G, store.d_v), dtype=torch.float32, device="cuda")
    sp = _lib.stream_ptr(stream)
    # q rows are addressed by absolute group id inside the kernel
    if margins is not None:  # + per (group, q-head) top-1 minus top-2 logit (gate input)
        assert margins.dtype == torch.float32 and margins.numel() == ng * G
        top2 = torch.empty((plan.n_slots + 1) * G, dtype=torch.float32, device="cuda")
        _lib.check(l.sphkv_ada_decode_margins(
            store.cptr_for(G), q.data_ptr(), G, plan.units.data_ptr(), plan.n_units,
            partials.data_ptr(), plan.slot_group.data_ptr(), plan.slot_begin.data_ptr(), ng,
            plan.ctl.data_ptr(), out.data_ptr(), int(plan.dynamic), top2.data_ptr(),
            margins.data_ptr(), plan.grid, sp))
        return out
    if logits is None:  # one launch: the last split of each group merges it in-kernel
        _lib.check(l.sphkv_ada_decode_fused(
            store.cptr_for(G), q.data_ptr(), G, plan.units.data_ptr(), plan.n_units,
            partials.data_ptr(), plan.slot_group.data_ptr(), plan.slot_begin.data_ptr(), ng,
            plan.ctl.data_ptr(), out.data_ptr(), int(plan.dynamic), plan.grid, sp))
        if plan.check_units:  # hand-made plans: surface an oversize unit (one sync)
            if int(plan.ctl[ng + 2].item()):
                plan.ctl[ng + 2] = 0
                raise RuntimeError("a decode unit exceeds the kernel's tile list "
                                   "(sphkv_unit_tile_cap); re-plan with plan_store")
        return out
    _lib.check(l.sphkv_ada_decode(store.cptr_for(G), q.data_ptr(), G, plan.units.data_ptr(),
                                  plan.n_units, partials.data_ptr(), _lib.ptr(logits),
                                  plan.dbg_offsets.data_ptr(), plan.grid, sp))
    _lib.check(l.sphkv_lse_merge(partials.data_ptr(), plan.slot_begin.data_ptr(), ng, G,
                                 store.d_v, out.data_ptr(), sp))
    return out


def ada_decode_state(store, q, plan: DecodePlan, *, state=None, partials=None, stream=None):
    """Fused decode of a (rank's page-range) plan whose in-kernel merge emits
    one partial STATE per planned group ([len(plan.group_ids), G*(d_v+2)]:
    log2-sum-exp, 1, normalized output) -- the operand of the all-gather and
    merge over ranks (plan.merge_gathered)."""
    import torch

    l = _lib.require_gpu()
    G = q.shape[-2]
    ng = len(plan.group_ids)
    if partials is None:
        partials = _partials(plan, G, store.d_v)
    if state is None:
        state = torch.empty((ng, G * (store.d_v + 2)), dtype=torch.float32, device="cuda")
    _lib.check(l.sphkv_ada_decode_state(
        store.cptr_for(G), q.data_ptr(), G, plan.units.data_ptr(), plan.n_units,
        partials.data_ptr(), plan.slot_group.data_ptr(), plan.slot_begin.data_ptr(), ng,
        plan.ctl.data_ptr(), state.data_ptr(), plan.grid, _lib.stream_ptr(stream)))
    return state


def dense_decode(dstore, q, plan: DecodePlan | None = None, *, out=None, partials=None,
                 stream=None, token_begin=0):
    """Dense bf16 paged decode (decode.py:63-69, 302-307); `token_begin` > 0
    attends only tokens >= token_begin (a sliding-window layer)."""
    import torch

    l = _lib.require_gpu()
    if plan is None:
        plan = plan_dense(dstore)
    G = q.shape[-2]
    if partials is None:
        partials = _partials(plan, G, dstore.d_v)
    ng = len(plan.group_ids)
    if out is None:
        out = torch.empty((ng * G, dstore.d_v), dtype=torch.float32, device="cuda")
    sp = _lib.stream_ptr(stream)
    _lib.check(l.sphkv_dense_decode_window(
        dstore.cptr, q.data_ptr(), G, plan.units.data_ptr(), plan.n_units, partials.data_ptr(),
        plan.slot_group.data_ptr(), plan.slot_begin.data_ptr(), ng, plan.ctl.data_ptr(),
        out.data_ptr(), int(plan.dynamic), int(token_begin), plan.grid, sp))
    return out


def lse_merge(partials, slot_begin, n_groups, G, d_v, out=None, stream=None):
    """Split-context merge of partial (m, l, acc) states (base-2 logit units)."""
    import torch

    l = _lib.require_gpu()
    if out is None:
        out = torch.empty((n_groups * G, d_v), dtype=torch.float32, device="cuda")
    _lib.check(l.sphkv_lse_merge(partials.data_ptr(), slot_begin.data_ptr(), n_groups, G, d_v,
                                 out.data_ptr(), _lib.stream_ptr(stream)))
    return out


# ---------------------------------------------------------------------------
# reference-shaped wrappers (numpy in / numpy out)
# ---------------------------------------------------------------------------

def attend_heads(store, layer, head, queries, seq=0):
    """All G query heads of one KV head: returns (logits [G, n], outputs [G, d_v])."""
    import torch

    queries = np.atleast_2d(np.asarray(queries, dtype=np.float64))
    G, d = queries.shape
    if d != store.d:
        raise ValueError(f"dimension mismatch: q has {d}, store {store.d}")
    if not (0 <= layer < store.layers and 0 <= head < store.heads):
        raise KeyError(f"unknown (layer, head) = {(layer, head)}")
    g = store._group(layer, head, seq)
    plan = plan_store(store, groups=[g], grid=8, units_per_cta=1)
    q = torch.zeros((store.groups, G, d), dtype=torch.float32, device="cuda")
    q[g] = torch.as_tensor(queries, dtype=torch.float32, device="cuda")
    n = int(plan.group_items[0])
    lg = torch.zeros(max(n, 1) * G, dtype=torch.float32, device="cuda")
    out = ada_decode(store, q, plan, logits=lg)
    logits = lg[: n * G].view(n, G).T.double().cpu().numpy()
    return logits, out.double().cpu().numpy()


def _query_vector(q, store, query_tier):
    q = np.asarray(q, dtype=np.float64)
    if query_tier is None or query_tier == 0:
        return q
    from . import codec

    s = codec.to_spherical(q)
    t = store.tiers.spec_for(query_tier)
    ang = codec.dequantize_angles(codec.quantize_angles(s.angles[None], t.angle_bits),
                                  t.angle_bits)[0]
    return s.radius * codec.angular_features(ang[None])[0]


def angle_logits(q, store, layer, head, query_tier=None) -> np.ndarray:
    """Compressed-domain logits (decode.py:175-192) from the device kernel."""
    qv = _query_vector(q, store, query_tier)
    if not np.any(qv):
        raise ValueError("query must be nonzero")
    logits, _ = attend_heads(store, layer, head, qv[None])
    store.meter_stream(layer, head)  # exactly the streamed header, code and value bytes
    return logits[0]


def _recon_stage(store, layer, head, stage_dtype="f32"):
    """Device reconstruction of one head's keys in pointer order (the staging
    write of the reconstruct-then-dot path); meters the streamed pages and the
    densification tax exactly as decode.py:195-217 does."""
    import torch

    l = _lib.require_gpu()
    pages = [(i, p.count) for i, p in store.stream_pages(layer, head)]  # meters reads
    live = [(i, c) for i, c in pages if c > 0]
    if not live:
        return None, []
    pids = np.array([i for i, _ in live], dtype=np.int32)
    counts = np.array([c for _, c in live], dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
    total = int(counts.sum())
    dt = {"f32": (torch.float32, _lib.F32), "f16": (torch.float16, _lib.F16)}[stage_dtype]
    stage = torch.empty((total, store.d), dtype=dt[0], device="cuda")
    pid_t = torch.as_tensor(pids, device="cuda")
    off_t = torch.as_tensor(off, device="cuda")
    _lib.check(l.sphkv_recon_keys(store.cptr, pid_t.data_ptr(), off_t.data_ptr(), len(pids),
                                  stage.data_ptr(), dt[1], _lib.stream_ptr()))
    tax = store.d * 2  # dense stage bytes per item, each direction (decode.py:208)
    store.meter.add_write("dense_k_write", total * tax)
    store.meter.add_read("dense_k_read", total * tax)
    return stage, [i for i, _ in live]


def _recon_dot(stage, q, d):
    """The dot's re-read of the staged rows on the device (sphkv_recon_dot):
    q [G, d] (or [d]) -> logits [n, G] fp32 (natural units)."""
    import torch

    l = _lib.require_gpu()
    q = np.atleast_2d(np.asarray(q, dtype=np.float64))
    qd = torch.as_tensor(q, dtype=torch.float32, device="cuda").contiguous()
    n = stage.shape[0]
    out = torch.empty((n, q.shape[0]), dtype=torch.float32, device="cuda")
    dt = _lib.F32 if stage.dtype == torch.float32 else _lib.F16
    _lib.check(l.sphkv_recon_dot(stage.data_ptr(), dt, n, d, qd.data_ptr(), q.shape[0],
                                 out.data_ptr(), _lib.stream_ptr()))
    return out


def recon_logits(q, store, layer, head) -> np.ndarray:
    """Reconstruct-then-dot negative control (decode.py:195-217): same numbers
    as angle_logits, plus the dense staging write and re-read (both kernels)."""
    q = np.asarray(q, dtype=np.float64)
    stage, _ = _recon_stage(store, layer, head)
    if stage is None:
        return np.empty(0)
    return _recon_dot(stage, q, store.d)[:, 0].double().cpu().numpy()


def dense_logits(q, keys) -> np.ndarray:
    """Reference dense logits keys @ q / sqrt(d) (decode.py:63-69), fp64 on
    the device (sphkv_dense_logits)."""
    import torch

    q = np.asarray(q, dtype=np.float64)
    keys = np.asarray(keys, dtype=np.float64)
    if keys.ndim != 2 or keys.shape[1] != q.shape[0]:
        raise ValueError(f"dimension mismatch: q has {q.shape[0]}, keys {keys.shape}")
    l = _lib.require_gpu()
    n, d = keys.shape
    if n == 0:
        return np.empty(0)
    qd = torch.as_tensor(q, device="cuda")
    kd = torch.as_tensor(np.ascontiguousarray(keys), device="cuda")
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(l.sphkv_dense_logits(qd.data_ptr(), kd.data_ptr(), n, d, out.data_ptr(),
                                    _lib.stream_ptr()))
    return out.cpu().numpy()


def stable_softmax(logits: np.ndarray) -> np.ndarray:
    z = logits - logits.max()
    w = np.exp(z)
    return w / w.sum()


def softmax_mix(logits, values) -> AttentionOutput:
    logits = np.asarray(logits, dtype=np.float64)
    if logits.size == 0:
        raise ValueError("empty logits")
    values = np.asarray(values, dtype=np.float64)
    if values.shape[0] != logits.shape[0]:
        raise ValueError("values not aligned with logits")
    w = stable_softmax(logits)
    return AttentionOutput(w, w @ values)


def _head_attend(path, store, layer, head, q, raw_keys=None, qfeat_pair=None):
    """(logits, output, n_items, dense_ref_logits) for one head (decode.py:291-355).

    Meters as the reference does, once per call: dense -- headers, dense
    key and value bytes (store.stream_dense); angle / recon -- header, code
    and value bytes of every listed page, recon adds the densification tax."""
    if path not in PATHS:
        raise ValueError(f"unknown path {path!r}")
    if path == "recon":
        stage, pids = _recon_stage(store, layer, head)
        if stage is None:
            return np.empty(0), np.zeros(store.d_v), 0, None
        lg = _recon_dot(stage, q, store.d)[:, 0].double().cpu().numpy()
        values = np.concatenate([store.pages[i].values for i in pids])
        return lg, softmax_mix(lg, values).output, lg.size, None
    if path == "dense":
        import torch

        if not (0 <= layer < store.layers and 0 <= head < store.heads):
            raise KeyError(f"unknown (layer, head) = {(layer, head)}")
        store.meter_dense_stream()
        if store.tokens == 0:
            return np.empty(0), np.zeros(store.d_v), 0, None
        g = (layer * store.heads) + head
        qv = torch.zeros((store.batch * store.layers * store.heads, 1, store.d),
                         dtype=torch.float32, device="cuda")
        qv[g, 0] = torch.as_tensor(np.asarray(q, dtype=np.float64), device="cuda")
        plan = plan_dense(store, groups=[g], grid=8, units_per_cta=1)
        out = dense_decode(store, qv, plan)
        lg = store.logits(g, qv[g])[:, 0].double().cpu().numpy()
        return lg, out[0].double().cpu().numpy(), lg.size, None
    if qfeat_pair is not None:
        r_q, qfeat = qfeat_pair
        qv = float(r_q) * np.asarray(qfeat, dtype=np.float64)
    else:
        qv = np.asarray(q, dtype=np.float64)
    logits, out = attend_heads(store, layer, head, qv[None])
    store.meter_stream(layer, head)  # header + code + value bytes, batched (decode.py:336-342)
    lg = logits[0]
    ref = None
    if raw_keys is not None and lg.size:
        toks = np.concatenate([store._token_ids(i, store.pages[i].count)
                               for i in store.pointer[(layer, head)] if store.pages[i].count])
        ref = np.asarray(raw_keys)[toks] @ np.asarray(q, dtype=np.float64) / math.sqrt(store.d)
    if lg.size == 0:
        return np.empty(0), np.zeros(store.d_v), 0, ref
    return lg, out[0], lg.size, ref


def logit_drift_bound(r_q, r_k, eps_r, eps_theta, d) -> float:
    if min(r_q, r_k, eps_r, eps_theta) < 0:
        raise ValueError("drift bound inputs must be nonnegative")
    return (r_q / math.sqrt(d)) * (r_k * eps_theta + eps_r + eps_r * eps_theta)
