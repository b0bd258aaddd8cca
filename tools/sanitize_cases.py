"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): pack, fused ADA decode (static + dynamic plans, gate
margins, h-byte tables), debug-logit decode + LSE merge, dense decode, SPHKV1
import, appends and one captured decode step with appends."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import synth

torch.cuda.set_device(0)
L, H, G, T, d = 2, 2, 4, 3000, 128
wl = synth.generate(1, L, H, G, T, d, seed=3)
tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in synth.PANEL_TIERS))
for k, t in enumerate(tiers.non_drop):
    tiers.eps_theta[t.id], tiers.eps_r[t.id] = 0.05 / (k + 1), 0.01 / (k + 1)
n = wl.groups * T
rng = np.random.default_rng(0)
tier = rng.choice([0, 1, 2, 3, 4, 5, 6], n, p=[0.1, 0.4, 0.1, 0.1, 0.1, 0.15, 0.05]).astype(np.int16)
radii = torch.empty(n, dtype=torch.float64, device="cuda")
from paper_2605_18856_b200 import _lib
_lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, d, radii.data_ptr(),
                                         _lib.stream_ptr()))
st = sk.PagedStore(tiers, L, H, d, d, 256, capacity_tokens=T, append_tokens=64)
sk.pack_device(st, keys=wl.keys.view(-1, d), radii=radii, values=wl.values.view(-1, d),
               z=(tier != 0).astype(np.int8), tier=tier, protect=np.zeros(n, np.uint8), tokens=T)
q = wl.queries
a = sk.ada_decode(st, q, sk.plan_store(st, grid=148, units_per_cta=1))
b = sk.ada_decode(st, q, sk.plan_store(st, grid=20, units_per_cta=3, dynamic=True))
m = torch.empty(st.groups * G, dtype=torch.float32, device="cuda")
c = sk.ada_decode(st, q, sk.plan_store(st, grid=148, units_per_cta=1), margins=m)
lg, out = sk.decode.attend_heads(st, 1, 1, q[3].double().cpu().numpy())
st.hbyte_tables = True
e = sk.ada_decode(st, q, sk.plan_store(st, grid=148, units_per_cta=1))
st.hbyte_tables = False
ds = sk.DenseStore(L, H, d, d, 256)
ds.bulk_load(wl.keys, wl.values)
f = sk.dense_decode(ds, q)
g = sk.dense_decode(ds, q, token_begin=T - 128)
blob = st.to_bytes()
st2 = sk.PagedStore.from_bytes(blob, tiers)
assert st2.to_bytes() == blob
stp = sk.DecodeStepper(st, G, np.ones((L, H)), np.full((L, H), 0.5), 40.0, lam=3e-5,
                       gate_cfg=sk.GateConfig(0.05, 0.5))
stp.capture()
for t in range(3):
    stp.step(q, torch.randn((st.groups, d), device="cuda"),
             torch.randn((st.groups, d), device="cuda").half(), T + t)
stp.finish()
torch.cuda.synchronize()
print("sanitize cases ok", float((a - b).abs().max()), float((a - c).abs().max()),
      float((a - e).abs().max()))
