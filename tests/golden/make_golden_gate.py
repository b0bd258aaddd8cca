"""Golden vectors for the decode-time gate, made by running the REAL reference
(read-only checkout) in the build container:
    python tests/golden/make_golden_gate.py
Writes tests/golden/golden_gate.npz: random (drift bound, margin) pairs with
the reference danger_score, and hysteresis traces of gate_step."""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sphkv import gate  # noqa: E402

rng = np.random.default_rng(11)
n = 2000
bound = np.abs(rng.standard_normal(n)) * rng.choice([0.01, 0.3, 3.0], n)
marg = np.abs(rng.standard_normal(n)) * rng.choice([0.001, 0.1, 2.0], n)
marg[rng.random(n) < 0.05] = np.inf
danger = np.array([gate.danger_score(float(b), float(m)) for b, m in zip(bound, marg)])
logits = rng.standard_normal((64, 37)) * 3
logits[5, :] = 1.25  # ties
margins = np.array([gate.margin(row) for row in logits])
margins_small = np.array([gate.margin(logits[0, :1]), gate.margin(logits[0, :0])])
cfg = gate.GateConfig(tau_drop=0.2, tau_prot=0.8)
steps, heads = 40, 16
trace_d = np.abs(rng.standard_normal((steps, heads))) * 0.7
modes = np.zeros((steps, heads), dtype=np.int64)
actions = np.zeros((steps, heads), dtype=np.int64)
code = {"compressible": 0, "held": 1, "protected": 2}
acode = {gate.ACTION_ALLOW: 0, gate.ACTION_HOLD: 1, gate.ACTION_PROTECT: 2}
for h in range(heads):
    st = gate.GateState()
    for t in range(steps):
        a, st = gate.gate_step(float(trace_d[t, h]), st, cfg)
        modes[t, h], actions[t, h] = code[st.mode], acode[a]
out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_gate.npz")
np.savez_compressed(out, bound=bound, marg=marg, danger=danger, logits=logits, margins=margins,
                    margins_small=margins_small, trace_d=trace_d, modes=modes, actions=actions,
                    tau=np.array([cfg.tau_drop, cfg.tau_prot]))
print("wrote", out)
