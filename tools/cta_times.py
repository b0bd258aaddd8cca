"""Per-CTA time spread of one c5 layer launch (needs a -DSPHKV_DBG_TIMING build)."""
import ctypes, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import _lib, plan as planmod

W = bench.build_workload("c5", dense=False, parity=False)
st, qall = W["st"], W["q"]
B, L, H, G, T, d, _ = bench.CONFIGS["c5"]
lib = _lib.lib()
import os
LAYERS = [int(x) for x in os.environ.get("CTA_LAYERS", "0,5").split(",")]
raw = {}
for l in LAYERS:
    groups = [(b * L + l) * H + h for b in range(B) for h in range(H)]
    p = planmod.plan_store(st, groups=groups, units_per_cta=1)
    out = torch.empty((len(groups) * G, d), dtype=torch.float32, device="cuda")
    for _ in range(3):
        sk.ada_decode(st, qall, p, out=out)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (2 * p.grid))()
    lib.sphkv_debug_cta_times.argtypes = [ctypes.c_void_p, ctypes.c_int]
    _lib.check(lib.sphkv_debug_cta_times(ctypes.addressof(buf), p.grid))
    t = np.array(buf, dtype=np.float64).reshape(-1, 2)
    t0 = t[:, 0].min()
    s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = e - s
    n, rows, plen, ptr = st._host()
    cost = planmod._page_cost(rows, st.d)
    u = p.units_host
    pc = np.array([cost[ptr[g, a:b]].sum() for g, a, b in zip(u["group"], u["ptr_begin"], u["ptr_end"])])
    ab = np.array([np.bincount(rows["abits"][ptr[g, a:b]], weights=rows["count"][ptr[g, a:b]], minlength=16)
                   for g, a, b in zip(u["group"], u["ptr_begin"], u["ptr_end"])])
    print(f"layer {l}: start max {s.max():.1f} us, end min/mean/max {e.min():.1f}/{e.mean():.1f}/{e.max():.1f} us, "
          f"dur min/max {dur.min():.1f}/{dur.max():.1f}")
    # time per unit vs predicted cost: ratio spread; residual by dominant tier
    ratio = dur[: len(pc)] / (pc / 1e6)
    print("   us per predicted us: min %.2f mean %.2f max %.2f" % (ratio.min(), ratio.mean(), ratio.max()))
    print("   predicted cost per CTA (ps): min %d mean %d max %d, n units %d grid %d" % (
        pc.min(), pc.mean(), pc.max(), len(pc), p.grid))
    print("   corr(dur, pred) = %.3f" % np.corrcoef(dur[: len(pc)], pc)[0, 1])
    # least-squares per-bit-width cost (us per item) from the CTA durations
    X = ab[:, [2, 4, 6, 7, 12]]
    coef, *_ = np.linalg.lstsq(X, dur[: len(pc)], rcond=None)
    print("   fitted us/item by bits 2,4,6,7,12:", np.round(coef * 1e3, 2), "(ns)")
    print("   dur by blockIdx%8:", [round(float(dur[np.arange(len(dur)) % 8 == r].mean()), 1) for r in range(8)])
    print("   dur by blockIdx<74:", round(float(dur[:74].mean()), 1), round(float(dur[74:].mean()), 1))
    for i in np.argsort(-dur)[:5]:
        print("   slow cta", i, "dur %.1f" % dur[i], "pred %.1f" % (pc[i] / 1e6), "items by bits",
              {b: int(ab[i][b]) for b in range(16) if ab[i][b]})
    for i in np.argsort(dur)[:3]:
        print("   fast cta", i, "dur %.1f" % dur[i], "pred %.1f" % (pc[i] / 1e6), "items by bits",
              {b: int(ab[i][b]) for b in range(16) if ab[i][b]})
    raw[f"dur{l}"] = dur
    raw[f"ab{l}"] = ab
    raw[f"pc{l}"] = pc
    raw[f"np{l}"] = np.array([b - a for a, b in zip(u["ptr_begin"], u["ptr_end"])])
if os.environ.get("CTA_OUT"):
    np.savez(os.environ["CTA_OUT"], **raw)
