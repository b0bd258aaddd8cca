"""Decode-time gate: the package's scalar and batched gate
against golden vectors produced by the real reference (tests/golden/
make_golden_gate.py, gate.py:50-74).  CPU only (torch CPU tensors)."""

import math

import numpy as np
import pytest
import torch

from paper_2605_18856_b200 import gate


def test_scalar_gate_matches_reference(golden):
    g = golden("gate")
    for b, m, want in zip(g["bound"], g["marg"], g["danger"]):
        assert gate.danger_score(float(b), float(m)) == want
    assert [gate.margin(r) for r in g["logits"]] == list(g["margins"])
    small = [gate.margin(g["logits"][0, :1]), gate.margin(g["logits"][0, :0])]
    assert small == list(g["margins_small"]) == [math.inf, math.inf]
    with pytest.raises(ValueError):
        gate.danger_score(-1.0, 1.0)
    with pytest.raises(ValueError):
        gate.GateConfig(tau_drop=0.5, tau_prot=0.5)


def test_batched_gate_matches_reference(golden):
    g = golden("gate")
    d = gate.danger_batch(torch.as_tensor(g["bound"]), torch.as_tensor(g["marg"]))
    np.testing.assert_allclose(d.numpy(), g["danger"], rtol=1e-15, atol=0)
    cfg = gate.GateConfig(tau_drop=float(g["tau"][0]), tau_prot=float(g["tau"][1]))
    mode = torch.ones(g["trace_d"].shape[1], dtype=torch.int64)  # GateState() = "held"
    for t in range(g["trace_d"].shape[0]):
        action, mode = gate.gate_step_batch(torch.as_tensor(g["trace_d"][t]), mode, cfg)
        assert np.array_equal(mode.numpy(), g["modes"][t])
        assert np.array_equal(action.numpy(), g["actions"][t])


def test_kv_head_danger_is_max_over_query_heads():
    m = torch.tensor([0.5, 0.1, math.inf, 2.0, 0.2, 0.3])
    d = gate.kv_head_danger(torch.tensor(0.1), m, 3)
    want = torch.stack([gate.danger_batch(torch.tensor(0.1), m[:3]).max(),
                        gate.danger_batch(torch.tensor(0.1), m[3:]).max()])
    assert torch.equal(d, want)
