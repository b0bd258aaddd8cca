"""Where a full decode step's time goes (c5): plain fused decode graph vs the
live decode (with / without gate margins) vs the whole DecodeStepper step."""
import sys
import torch
sys.path.insert(0, ".")
import bench
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import _lib, synth
from paper_2605_18856_b200.gate import GateConfig

W = bench.build_workload("c5", parity=False, dense=False)
st, q = W["st"], W["q"]
G, d, T = 4, 128, 131072
l = _lib.require_gpu()


def timed(fn, n=20):
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


stp = sk.DecodeStepper(st, G, W["u_hat"], W["s_hat"], W["r_q"], lam=synth.PANEL_LAMBDA,
                       omega=synth.PANEL_OMEGA[2], gate_cfg=GateConfig(0.05, 0.5))
stp.q.copy_(q.view_as(stp.q))


def live(s, margins=True, flags0=_lib.LIVE_AFTER_MUTATION):
    cp = st.cptr_for(G)
    for i, (p, part, t2) in enumerate(zip(stp.plans, stp.parts, stp.top2)):
        flags = _lib.LIVE_ABS_ROWS | (flags0 if i == 0 else 0)
        _lib.check(l.sphkv_ada_decode_live(
            cp, stp.q.data_ptr(), G, p.units.data_ptr(), p.n_units, part.data_ptr(),
            p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids), p.ctl.data_ptr(),
            stp.out.data_ptr(), t2.data_ptr() if margins else None,
            stp.margins.data_ptr() if margins else None, flags, p.grid, s.cuda_stream))


def fused(s):
    cp = st.cptr_for(G)
    for p, part in zip(stp.plans, stp.parts):
        out = torch.empty((len(p.group_ids), G, d), device="cuda") if False else stp.out
        _lib.check(l.sphkv_ada_decode_fused(
            cp, stp.q.data_ptr(), G, p.units.data_ptr(), p.n_units, part.data_ptr(),
            p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids), p.ctl.data_ptr(),
            stp.out.data_ptr(), 0, p.grid, s.cuda_stream))


print("fused (plan order rows)      %.3f ms" % timed(fused))
print("live, margins                %.3f ms" % timed(lambda s: live(s, True)))
print("live, no margins             %.3f ms" % timed(lambda s: live(s, False)))
print("live, margins, PDL on all    %.3f ms" % timed(lambda s: live(s, True, 0)))
print("DecodeStepper step           %.3f ms" % timed(lambda s: stp._launch(s)))
print("DecodeStepper step w/o decode %.3f ms" % timed(lambda s: (
    _lib.check(l.sphkv_decode_gate(st.cptr, stp.k_new.data_ptr(), _lib.F32, stp.q.data_ptr(), G,
               stp.margins.data_ptr(), stp.u_hat.data_ptr(), stp.s_hat.data_ptr(), stp.r_q,
               stp.omega, 1.0, 1.0, stp.lam, 1, 0.05, 0.5, 1.0, stp.mode.data_ptr(),
               stp.tier.data_ptr(), stp.prot.data_ptr(), stp.danger.data_ptr(), s.cuda_stream)))))
