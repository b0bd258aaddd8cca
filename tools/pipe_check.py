"""Pipelined unit transitions (SPHKV_PIPE=1, k_ada_decode_pipe) vs the
standard kernel body on the same pages and plans: outputs must agree (same
tile math, same merge order) for static one-unit, tail-piece and dynamic
multi-unit plans; times per launch with CUDA events."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import plan as planmod

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
W = bench.build_workload(cfg, dense=False, parity=False)
st, qall = W["st"], W["q"]
B, L, H, G, T, d, _ = bench.CONFIGS[cfg]


def run(plan, pipe, it=20):
    os.environ["SPHKV_PIPE"] = "1" if pipe else "0"
    out = torch.empty((len(plan.group_ids) * G, st.d_v), dtype=torch.float32, device="cuda")
    for _ in range(3):
        sk.ada_decode(st, qall, plan, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        sk.ada_decode(st, qall, plan, out=out)
    b.record()
    torch.cuda.synchronize()
    return out.clone(), a.elapsed_time(b) / it * 1e3


worst = 0.0
for l in (0, 7):
    groups = [(b * L + l) * H + h for b in range(B) for h in range(H)]
    ref = None
    for name, kw in [("static", dict(units_per_cta=1)),
                     ("tail0.1", dict(units_per_cta=1, tail=0.1)),
                     ("tail0.2", dict(units_per_cta=1, tail=0.2)),
                     ("tail0.3x3", dict(units_per_cta=1, tail=0.3, tail_pieces=3)),
                     ("upc2dyn", dict(units_per_cta=2, dynamic=True)),
                     ("upc3dyn", dict(units_per_cta=3, dynamic=True))]:
        p = planmod.plan_store(st, groups=groups, **kw)
        o0, t0 = run(p, False)
        o1, t1 = run(p, True)
        if ref is None:
            ref = o0
        e01 = float((o1 - o0).abs().max() / o0.abs().max())
        eref = float((o1 - ref).abs().max() / ref.abs().max())
        worst = max(worst, e01, eref)
        print(f"layer {l} {name:9s} units {p.n_units:4d}: std {t0:6.1f} us  pipe {t1:6.1f} us  "
              f"|pipe-std| {e01:.2e}  |pipe-static std| {eref:.2e}", flush=True)
print("worst rel diff", worst)
assert worst < 1e-5, worst
