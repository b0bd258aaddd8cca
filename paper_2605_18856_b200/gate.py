"""Decode-time stability gate (drop-in for sphkv.gate, pkg/src/sphkv/gate.py:1-74).

The scalar API keeps the reference's names and semantics (`margin`,
`danger_score`, `gate_step`, `GateConfig`, `GateState`).  The batched forms run
the same rules on device tensors for every (seq, layer, kv-head) at once: the
margins come out of the decode kernel as a by-product
(`decode.ada_decode(..., margins=...)`, top-1 minus top-2 logit per query head
over all of the head's items), so a decode step's gate costs no extra pass over
the KV pages.  GQA (the reference has one query per head): a KV head's danger
is the max over its G query heads (the conservative choice).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DANGER_CLAMP = 10.0          # gate.py:24
_MARGIN_EPS = 1e-9           # gate.py:25

ACTION_PROTECT = "tier_up_or_protect"
ACTION_ALLOW = "allow_downtier"
ACTION_HOLD = "hold"

MODES = ("compressible", "held", "protected")  # batched mode codes 0, 1, 2


@dataclass(frozen=True)
class GateConfig:
    tau_drop: float
    tau_prot: float
    alpha: float = 1.0

    def __post_init__(self):
        if not self.tau_drop < self.tau_prot:
            raise ValueError("hysteresis needs tau_drop < tau_prot strictly")
        if self.alpha <= 0:
            raise ValueError("alpha must be positive")


@dataclass(frozen=True)
class GateState:
    mode: str = "held"
    last_danger: float = 0.0


def margin(logits) -> float:
    """Top-1 minus top-2 logit; +inf when fewer than two candidates (gate.py:50-56)."""
    logits = np.asarray(logits, dtype=np.float64)
    if logits.size < 2:
        return math.inf
    top2 = np.partition(logits, -2)[-2:]
    return float(top2[1] - top2[0])


def danger_score(drift_bound: float, margin_value: float) -> float:
    """Predicted drift over local margin, clamped to [0, 10] (gate.py:59-65)."""
    if drift_bound < 0 or margin_value < 0:
        raise ValueError("danger inputs must be nonnegative")
    if math.isinf(margin_value):
        return 0.0
    return min(drift_bound / (margin_value + _MARGIN_EPS), DANGER_CLAMP)


def gate_step(d_t: float, state: GateState, cfg: GateConfig):
    """One hysteretic transition; in-band danger holds the previous mode (gate.py:68-74)."""
    if d_t >= cfg.tau_prot:
        return ACTION_PROTECT, GateState("protected", d_t)
    if d_t <= cfg.tau_drop:
        return ACTION_ALLOW, GateState("compressible", d_t)
    return ACTION_HOLD, GateState(state.mode, d_t)


def danger_batch(drift_bound, margins):
    """danger_score over tensors (any shape, broadcast); margins may be +inf."""
    import torch

    if bool((drift_bound < 0).any()) or bool((margins < 0).any()):
        raise ValueError("danger inputs must be nonnegative")
    d = torch.clamp(drift_bound / (margins + _MARGIN_EPS), max=DANGER_CLAMP)
    return torch.where(torch.isinf(margins), torch.zeros_like(d), d)


def gate_step_batch(danger, mode, cfg: GateConfig):
    """gate_step for every head at once: returns (action codes, new modes).
    mode/new mode codes index MODES; action codes 0 = allow, 1 = hold,
    2 = protect."""
    import torch

    prot = danger >= cfg.tau_prot
    allow = (~prot) & (danger <= cfg.tau_drop)
    new_mode = torch.where(prot, torch.full_like(mode, 2),
                           torch.where(allow, torch.zeros_like(mode), mode))
    action = torch.where(prot, torch.full_like(mode, 2),
                         torch.where(allow, torch.zeros_like(mode), torch.ones_like(mode)))
    return action, new_mode


def kv_head_danger(drift_bound, margins, G: int):
    """Per KV head danger from per query-head margins [groups * G]: the max
    over the G query heads of each group (GQA mapping, module docstring)."""
    d = danger_batch(drift_bound, margins.view(-1, G))
    return d.max(dim=-1).values
