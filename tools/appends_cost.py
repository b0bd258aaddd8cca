"""Kernel time breakdown of one full decode step with appends (c5 workload):
torch.profiler (CUPTI) over a few DecodeStepper steps, per kernel name."""
import sys
import collections
import torch
sys.path.insert(0, ".")
import bench
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import synth
from paper_2605_18856_b200.gate import GateConfig

W = bench.build_workload("c5", parity=False, dense=False)
st, q = W["st"], W["q"]
G, d, T = 4, 128, 131072
stp = sk.DecodeStepper(st, G, W["u_hat"], W["s_hat"], W["r_q"], lam=synth.PANEL_LAMBDA,
                       omega=synth.PANEL_OMEGA[2], gate_cfg=GateConfig(0.05, 0.5))
gen = torch.Generator(device="cuda")
gen.manual_seed(1)
kn = torch.randn((20, st.groups, d), generator=gen, device="cuda") / d ** 0.5 + 0.1
vn = torch.randn((20, st.groups, d), generator=gen, device="cuda").half()
stp.capture()
for t in range(3):
    stp.step(q, kn[t], vn[t], T + t)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for t in range(5):
        stp.step(None, kn[3 + t], vn[3 + t], T + 3 + t)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        agg[e.name[:60]][0] += 1
        agg[e.name[:60]][1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us / 5:9.1f} us/step  {n / 5:5.1f} launches/step  {k}")
