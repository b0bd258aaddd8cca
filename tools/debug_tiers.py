"""Per-tier ADA logit error vs the oracle (debug aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2605_18856_b200 as sk
from oracle import sphkv_oracle as O

rng = np.random.default_rng(0)
for d, P, T in ((8, 32, 100), (128, 256, 600)):
    for B in (1, 2, 3, 4, 5, 7, 8, 12, 15):
        tl = [(0, 0, 0, 0), (1, B, 8, 0)]
        tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
        keys = rng.standard_normal((1, 1, T, d))
        vals = rng.standard_normal((1, 1, T, d)).astype(np.float16).astype(np.float64)
        r, ang = O.encode_batch(keys.reshape(-1, d))
        r, ang = r.reshape(1, 1, T), ang.reshape(1, 1, T, d - 1)
        tier = np.ones((1, 1, T), np.int16)
        z = tier.astype(np.int8)
        prot = np.zeros((1, 1, T), bool)
        st = sk.pack_pages_arrays(sk.TierAssignment(z, tier, prot), r, ang, vals, tiers, P)
        ost = O.pack_pages(tl, z, tier, prot, r, ang, vals, P)
        q = rng.standard_normal((4, d)) * 3
        lg, out = sk.decode.attend_heads(st, 0, 0, q)
        rq, qf = O.query_features(q)
        errs = []
        for g in range(4):
            wl, wo = O.head_attend(ost, 0, 0, rq[g], qf[g])
            e = np.abs(lg[g] - wl) / np.maximum(1, np.abs(wl))
            errs.append(e.max())
            if g == 0 and e.max() > 1e-3:
                bad = np.nonzero(e > 1e-3)[0]
                print("   bad items", bad[:20], "of", len(e))
        print(f"d={d} P={P} B={B:2d} max logit err {max(errs):.3e}", flush=True)
