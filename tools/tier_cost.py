"""Per-tier cost of k_ada_decode: one layer of 8 KV heads x 128K tokens (G=4,
d=128, P=256), every item at one panel tier.  Prints us per launch, ns per
item and achieved GB/s (algorithmic bytes) per tier, plus the dense kernel."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import _lib, synth

T, H, G, d = int(sys.argv[1]) if len(sys.argv) > 1 else 131072, 8, 4, 128
wl = synth.generate(1, 1, H, G, T, d, seed=0)
n = wl.groups * T
radii = torch.empty(n, dtype=torch.float64, device="cuda")
_lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, d, radii.data_ptr(),
                                         _lib.stream_ptr()))
tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in synth.PANEL_TIERS))


def timeit(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


for t in tiers.non_drop:
    st = sk.PagedStore(tiers, 1, H, d, d, 256, capacity_tokens=T)
    tier = torch.full((n,), t.id, dtype=torch.int16, device="cuda")
    sk.pack_device(st, keys=wl.keys.view(-1, d), radii=radii, values=wl.values.view(-1, d),
                   z=torch.ones(n, dtype=torch.int8, device="cuda"), tier=tier,
                   protect=torch.zeros(n, dtype=torch.uint8, device="cuda"), tokens=T)
    plan = sk.plan_store(st, units_per_cta=1)
    out = torch.empty((H * G, d), dtype=torch.float32, device="cuda")
    parts = sk.decode._partials(plan, G, d)
    us = timeit(lambda: sk.ada_decode(st, wl.queries, plan, out=out, partials=parts))
    by = st.stream_bytes_total()
    print(f"tier {t.id} (b_theta={t.angle_bits:2d}): {us:8.1f} us  {us * 1e3 / n:6.3f} ns/item  "
          f"{by / us / 1e3:7.1f} GB/s  bytes/item {by / n:6.1f}", flush=True)
    del st
ds = sk.DenseStore(1, H, d, d, 256)
ds.bulk_load(wl.keys, wl.values)
dp = sk.plan_dense(ds)
out = torch.empty((H * G, d), dtype=torch.float32, device="cuda")
us = timeit(lambda: sk.dense_decode(ds, wl.queries, dp, out=out))
print(f"dense        : {us:8.1f} us  {us * 1e3 / n:6.3f} ns/item  "
      f"{ds.stream_bytes_total() / us / 1e3:7.1f} GB/s", flush=True)
