"""Decode steps with appends on the device (the decode loop of decode.py:415-498).

Per step, for every (seq, layer, kv-head) group of a store:

1. attention over the group's CURRENT pages -- the fused ADA decode with the
   gate margins (top-1 minus top-2 logit per query head) as a by-product
   (`sphkv_ada_decode_live`: open-ended units reach pages appended by earlier
   steps, so one plan serves every step);
2. the append decision for the step's new key -- best tier
   (score_and_best_tier, controller.py:181-198) and, with a gate config, the
   hysteretic decode-time gate on the margins (gate.py:59-74; a protected head
   appends at the max tier with its protect flag) -- `sphkv_decode_gate`;
3. the append itself (store.py:249-274) -- `sphkv_append` encodes the key,
   opens pages by the reference rule and writes codes, values, flags.

All three are device launches on one stream with no host round trip, so a
step is captured once as a CUDA graph and replayed (`capture()` / `step()`).
GQA: a reference head is a KV head; its danger is the max over its G query
heads.  The new key's radius is the batched path's pairwise norm everywhere
(decode.py:457), as in the prefill encoder.  The toy LM that drives the
reference rollout's queries and new K/V is outside the hot path: the caller
supplies each step's queries and new keys/values.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .plan import plan_store

MODE_COMPRESSIBLE, MODE_HELD, MODE_PROTECTED = 0, 1, 2


class DecodeStepper:
    """Device decode steps with appends over one PagedStore.

    u_hat, s_hat: controller features per group ([store.groups] fp64, or
    [layers, heads] for one sequence); r_q, lam, alpha_*: as in
    ControllerFeatures / score_and_best_tier; omega: the weight of newly
    generated tokens (ControllerFeatures.omega_of for token >= prefill, i.e.
    the recent-segment weight).  gate_cfg: GateConfig or None (no gate)."""

    def __init__(self, store, G, u_hat, s_hat, r_q, *, lam=0.0, omega=1.0, alpha_theta=1.0,
                 alpha_r=1.0, gate_cfg=None, per_layer=True, grid=148, open_reserve_tiles=16.0):
        import torch

        self.l = _lib.require_gpu()
        self.st, self.G = store, G
        d, dv, groups = store.d, store.d_v, store.groups
        self.r_q, self.lam, self.omega = float(r_q), float(lam), float(omega)
        self.alpha_theta, self.alpha_r = float(alpha_theta), float(alpha_r)
        self.gate = gate_cfg
        dev = "cuda"
        self.u_hat = torch.as_tensor(np.asarray(u_hat, np.float64).reshape(-1), device=dev)
        self.s_hat = torch.as_tensor(np.asarray(s_hat, np.float64).reshape(-1), device=dev)
        if self.u_hat.numel() != groups or self.s_hat.numel() != groups:
            raise ValueError("u_hat / s_hat need one value per (seq, layer, head) group")
        if per_layer:  # one launch per layer (a model's attention runs layer by layer)
            L, H = store.layers, store.heads
            lists = [[(b * L + l) * H + h for b in range(store.batch) for h in range(H)]
                     for l in range(L)]
        else:
            lists = [list(range(groups))]
        # the last unit of a group also decodes the pages the steps append (a
        # partly filled page per tier in use): it gets a few tiles less prefill
        self.plans = [plan_store(store, groups=g, grid=grid, units_per_cta=1, open_end=True,
                                 open_reserve_tiles=open_reserve_tiles) for g in lists]
        self.q = torch.zeros((groups, G, d), dtype=torch.float32, device=dev)
        self.k_new = torch.zeros((groups, d), dtype=torch.float32, device=dev)
        self.v_new = torch.zeros((groups, dv), dtype=torch.float16, device=dev)
        self.token = torch.zeros(groups, dtype=torch.int64, device=dev)
        F = G * (dv + 2)
        self.parts = [torch.empty((p.n_slots + 1) * F, dtype=torch.float32, device=dev)
                      for p in self.plans]
        self.top2 = [torch.empty((p.n_slots + 1) * G, dtype=torch.float32, device=dev)
                     for p in self.plans]
        self.margins = torch.full((groups * G,), float("inf"), dtype=torch.float32, device=dev)
        self.out = torch.empty((groups, G, dv), dtype=torch.float32, device=dev)
        self.mode = torch.full((groups,), MODE_HELD, dtype=torch.int8, device=dev)
        self.tier = torch.zeros(groups, dtype=torch.int16, device=dev)
        self.prot = torch.zeros(groups, dtype=torch.uint8, device=dev)
        self.danger = torch.zeros(groups, dtype=torch.float32, device=dev)
        self.ws = torch.empty(self.l.sphkv_append_workspace_bytes(groups), dtype=torch.uint8,
                              device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)  # sticky over steps
        self.graph = None
        store.cptr_for(G)  # build the table variant the launches use (before any capture)

    # -- the step's device work -------------------------------------------------
    def _launch(self, stream):
        import torch

        l, st, G = self.l, self.st, self.G
        sp = stream.cuda_stream
        cp = st.cptr_for(G)
        for i, (p, part, t2) in enumerate(zip(self.plans, self.parts, self.top2)):
            # the first launch follows the previous step's append (no early
            # page-table reads); the others overlap their predecessor (PDL)
            flags = _lib.LIVE_ABS_ROWS | (_lib.LIVE_AFTER_MUTATION if i == 0 else 0)
            _lib.check(l.sphkv_ada_decode_live(
                cp, self.q.data_ptr(), G, p.units.data_ptr(), p.n_units, part.data_ptr(),
                p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids),
                p.ctl.data_ptr(), self.out.data_ptr(), t2.data_ptr(), self.margins.data_ptr(),
                flags, p.grid, sp))
        g = self.gate
        _lib.check(l.sphkv_decode_gate(
            st.cptr, self.k_new.data_ptr(), _lib.F32, self.q.data_ptr(), G,
            self.margins.data_ptr(), self.u_hat.data_ptr(), self.s_hat.data_ptr(), self.r_q,
            self.omega, self.alpha_theta, self.alpha_r, self.lam, int(g is not None),
            float(g.tau_drop) if g else 0.0, float(g.tau_prot) if g else 1.0,
            float(g.alpha) if g else 1.0, self.mode.data_ptr(), self.tier.data_ptr(),
            self.prot.data_ptr(), self.danger.data_ptr(), sp))
        _lib.check(l.sphkv_append(
            st.cptr, self.k_new.data_ptr(), _lib.F32, None, None, self.v_new.data_ptr(),
            self.tier.data_ptr(), self.prot.data_ptr(), self.token.data_ptr(), None,
            self.ws.data_ptr(), sp))
        torch.maximum(self.err, self.ws[:4].view(torch.int32), out=self.err)

    def capture(self, stream=None):
        """Capture one step as a CUDA graph (replayed by step())."""
        import torch

        stream = stream or torch.cuda.Stream()
        self._stream = stream
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            self._launch(stream)
        self.graph = g
        return g

    def step(self, q=None, k_new=None, v_new=None, token_id=None, stream=None):
        """One decode token: q [groups, G, d] fp32, k_new [groups, d], v_new
        [groups, d_v], token_id (int or [groups]); inputs may be host or device
        tensors.  Returns the attention outputs [groups, G, d_v] (device)."""
        import torch

        caller = torch.cuda.current_stream()
        stream = stream or getattr(self, "_stream", None) or caller
        if stream != caller:
            stream.wait_stream(caller)  # inputs the caller produced on its stream
        with torch.cuda.stream(stream):
            if q is not None:
                self.q.copy_(torch.as_tensor(q).view_as(self.q), non_blocking=True)
            if k_new is not None:
                self.k_new.copy_(torch.as_tensor(k_new).view_as(self.k_new), non_blocking=True)
            if v_new is not None:
                self.v_new.copy_(torch.as_tensor(v_new).view_as(self.v_new), non_blocking=True)
            if token_id is not None:
                if isinstance(token_id, int):
                    self.token.fill_(token_id)
                else:
                    self.token.copy_(torch.as_tensor(token_id).view_as(self.token))
            if self.graph is not None:
                self.graph.replay()
            else:
                self._launch(stream)
        if stream != caller:
            caller.wait_stream(stream)  # results are ordered before the caller's next work
        return self.out

    def finish(self):
        """Synchronize, surface append errors (pool / pointer-list capacity,
        unknown tier) and decode units that outgrew the tile list, and refresh
        the store's host views and table placement."""
        import torch

        torch.cuda.synchronize()
        err = int(self.err.item())
        oversize = any(int(p.ctl[len(p.group_ids) + 2].item()) for p in self.plans)
        self.st._invalidate()
        if oversize:
            raise RuntimeError("a live decode unit outgrew the kernel's tile list "
                               "(sphkv_unit_tile_cap); build a new DecodeStepper")
        if err == 3:
            raise RuntimeError("store pool exhausted during decode appends")
        if err == 4:
            raise RuntimeError("pointer list capacity exceeded during decode appends")
        if err == 5:
            raise KeyError("unknown tier id in append")
        self.st._refresh_lut()
