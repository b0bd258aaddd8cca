"""Generate golden vectors by running the REAL reference (read-only checkout).

Run in the build container only (the reference does not exist on the GPU
box):   python tests/golden/make_golden.py
Writes tests/golden/golden_*.npz; tests/test_oracle_golden.py replays them
against oracle/sphkv_oracle.py, and the -m gpu tests replay them against the
CUDA path.  Everything is seeded; re-running reproduces the files.
"""

from __future__ import annotations

import io
import math
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from sphkv import codec, decode, store as rstore  # noqa: E402
from sphkv.bitpack import pack_bits  # noqa: E402
from sphkv.codec import SphericalKey, TierSpec, TierTable  # noqa: E402
from sphkv.controller import (ControllerFeatures, TierAssignment,  # noqa: E402
                              allocate_greedy, downtier_before_drop,
                              full_best_tier_assignment, score_and_best_tier,
                              score_states, StateId)

OUT = os.path.dirname(os.path.abspath(__file__))

PANEL = ((0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 6, 8, 8), (4, 7, 8, 8),
         (5, 12, 14, 8), (6, 15, 16, 8))


def table(tiers, eps=None):
    t = TierTable(tuple(TierSpec(*x) for x in tiers))
    if eps is not None:
        for tid, (a, b) in eps.items():
            t.eps_theta[tid] = a
            t.eps_r[tid] = b
    return t


def pair_norm(k):
    return np.linalg.norm(k, axis=1)


def gen_codec():
    rng = np.random.default_rng(1234)
    out = {}
    for d in (2, 3, 8, 64, 128):
        n = 256
        k = rng.standard_normal((n, d))
        k[:, : max(d // 4, 1)] *= 0.01          # near-polar angles
        k[0] = 0.0                              # zero vector convention
        k[1] = 0.0
        k[1, 0] = -2.0                          # negative lead, zero tail
        k[2] = 0.0
        k[2, d - 1] = 1.5                       # last-axis vector
        k[3] = -k[4]
        r = pair_norm(k)
        ang = codec.angles_from_unit(k / (r[:, None] + 1e-12))
        ang[r == 0.0] = 0.0
        out[f"d{d}_keys"] = k
        out[f"d{d}_radii"] = r
        out[f"d{d}_angles"] = ang
        for b in (1, 2, 4, 6, 7, 8, 12, 15, 16):
            out[f"d{d}_codes_b{b}"] = codec.quantize_angles(ang, b).astype(np.uint16)
        # dequantized angles and features of a 4-bit tier (decode-side rows)
        deq = codec.dequantize_angles(out[f"d{d}_codes_b4"].astype(np.uint64), 4)
        out[f"d{d}_deq_b4"] = deq
        out[f"d{d}_feat_b4"] = codec.angular_features(deq)
        # scalar radius quantizer (append path) at a few scales
        scales = r.max() * np.array([1.0, 1.25, 3.0])
        rc = np.array([[codec.quantize_radius(float(x), float(s), br) for x in r]
                       for s in scales for br in (4, 8, 14)], dtype=np.int64)
        out[f"d{d}_rscales"] = scales
        out[f"d{d}_rcodes_append"] = rc
    np.savez_compressed(os.path.join(OUT, "golden_codec.npz"), **out)


def gen_bitpack():
    rng = np.random.default_rng(99)
    out = {}
    for bits in list(range(1, 17)) + [20, 31, 53]:
        n = int(rng.integers(0, 300))
        codes = rng.integers(0, 1 << bits, size=n, dtype=np.uint64)
        out[f"b{bits}_codes"] = codes
        out[f"b{bits}_stream"] = pack_bits(codes, bits)
    np.savez_compressed(os.path.join(OUT, "golden_bitpack.npz"), **out)


def _store_case(rng, L, H, T, d, dv, P, tiers, drop_frac, prot_frac):
    keys = rng.standard_normal((L, H, T, d))
    keys *= np.abs(rng.normal(1.0, 0.3, size=(L, H, T, 1)))
    vals = rng.standard_normal((L, H, T, dv)).astype(np.float16).astype(np.float64)
    flat = keys.reshape(-1, d)
    r = pair_norm(flat)
    ang = codec.angles_from_unit(flat / (r[:, None] + 1e-12)).reshape(L, H, T, d - 1)
    r = r.reshape(L, H, T)
    tier_ids = [t[0] for t in tiers[1:]]
    tier = rng.choice(tier_ids, size=(L, H, T)).astype(np.int16)
    drop = rng.random((L, H, T)) < drop_frac
    tier[drop] = 0
    z = (tier != 0).astype(np.int8)
    prot = (rng.random((L, H, T)) < prot_frac) & (z == 1)
    tier[prot] = tiers[-1][0]
    asg = TierAssignment(z, tier, prot)
    return keys, vals, r, ang, asg


def _dump_store(prefix, st, out):
    out[prefix + "n_pages"] = np.int64(len(st.pages))
    meta = np.array([[p.tier.id, p.layer, p.head, p.count] for p in st.pages],
                    dtype=np.int64).reshape(-1, 4)
    out[prefix + "meta"] = meta
    out[prefix + "scales"] = np.array([p.radius_scale for p in st.pages])
    ptr = []
    for l in range(st.layers):
        for h in range(st.heads):
            ptr.append(np.asarray(st.pointer[(l, h)], dtype=np.int64))
    out[prefix + "ptr_len"] = np.array([len(x) for x in ptr], dtype=np.int64)
    out[prefix + "ptr"] = np.concatenate(ptr) if ptr else np.zeros(0, np.int64)
    a_streams = [p.angle_stream(st.d) for p in st.pages]
    r_streams = [p.radius_stream() for p in st.pages]
    out[prefix + "astream_len"] = np.array([len(a) for a in a_streams], dtype=np.int64)
    out[prefix + "astream"] = (np.concatenate(a_streams) if a_streams
                               else np.zeros(0, np.uint8))
    out[prefix + "rstream_len"] = np.array([len(a) for a in r_streams], dtype=np.int64)
    out[prefix + "rstream"] = (np.concatenate(r_streams) if r_streams
                               else np.zeros(0, np.uint8))
    out[prefix + "token_ids"] = (np.concatenate([p.token_ids[: p.count] for p in st.pages])
                                 if st.pages else np.zeros(0, np.int64))
    br = st.resident_breakdown()
    out[prefix + "resident"] = np.array([br.payload_bytes, br.header_bytes, br.ptr_bytes,
                                         br.tag_bytes, br.prot_bytes, br.frag_bytes,
                                         br.total], dtype=np.int64)
    out[prefix + "stream_bytes"] = np.array(
        [st.expected_stream_bytes(l, h) for l in range(st.layers) for h in range(st.heads)],
        dtype=np.int64)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "s.bin")
        st.to_file(path)
        with open(path, "rb") as f:
            out[prefix + "sphkv1"] = np.frombuffer(f.read(), dtype=np.uint8)


def gen_store_attend():
    rng = np.random.default_rng(2024)
    out = {}
    cases = [
        # name, L, H, T, d, dv, P, tiers, drop, prot, G
        ("small", 2, 2, 300, 8, 8, 32, ((0, 0, 0, 0), (1, 4, 8, 0), (2, 8, 8, 8)), 0.2, 0.05, 2),
        ("panel64", 1, 2, 400, 64, 64, 64, PANEL, 0.1, 0.02, 4),
        ("panel128", 1, 2, 300, 128, 128, 256, PANEL, 0.05, 0.01, 4),
        ("odd", 1, 1, 77, 5, 3, 32, ((0, 0, 0, 0), (1, 3, 5, 2), (2, 9, 11, 0)), 0.3, 0.0, 3),
    ]
    for name, L, H, T, d, dv, P, tiers, drop, prot, G in cases:
        p = name + "_"
        tt = table(tiers)
        keys, vals, r, ang, asg = _store_case(rng, L, H, T, d, dv, P, tiers, drop, prot)
        st = rstore.pack_pages_arrays(asg, r, ang, vals, tt, P)
        out[p + "dims"] = np.array([L, H, T, d, dv, P, G], dtype=np.int64)
        out[p + "tiers"] = np.array(tiers, dtype=np.int64)
        out[p + "keys"] = keys
        out[p + "values"] = vals
        out[p + "radii"] = r
        out[p + "angles"] = ang
        out[p + "z"] = asg.z
        out[p + "tier"] = asg.tier
        out[p + "protected"] = asg.protected
        _dump_store(p + "pack_", st, out)
        # attend: G queries per (l, h) through the reference's angle branch
        q = rng.standard_normal((L, H, G, d)) * 3.0
        qn = np.linalg.norm(q, axis=-1)
        units = (q / (qn[..., None] + 1e-12)).reshape(-1, d)
        qfeat = codec.angular_features(codec.angles_from_unit(units)).reshape(L, H, G, d)
        logits, outs = [], []
        for l in range(L):
            for h in range(H):
                for g in range(G):
                    lg, o, n, _ = decode._head_attend(
                        "angle", st, l, h, q[l, h, g],
                        qfeat_pair=(float(qn[l, h, g]), qfeat[l, h, g]))
                    logits.append(lg)
                    outs.append(o)
        out[p + "q"] = q
        out[p + "logits_len"] = np.array([len(x) for x in logits], dtype=np.int64)
        out[p + "logits"] = np.concatenate(logits)
        out[p + "outputs"] = np.stack(outs)
        # appends on top of the packed store (store.py:249-274)
        n_app = 40
        ak = rng.standard_normal((n_app, d)) * np.abs(rng.normal(1.0, 0.8, (n_app, 1)))
        ak[5] *= 10.0  # forces a new page (radius above scale)
        ar = pair_norm(ak)
        aang = codec.angles_from_unit(ak / (ar[:, None] + 1e-12))
        av = rng.standard_normal((n_app, dv)).astype(np.float16).astype(np.float64)
        al = rng.integers(0, L, n_app)
        ah = rng.integers(0, H, n_app)
        at = rng.choice([t[0] for t in tiers], n_app)
        ap = rng.random(n_app) < 0.1
        for i in range(n_app):
            st.append_item(int(al[i]), int(ah[i]), SphericalKey(float(ar[i]), aang[i]),
                           av[i], int(at[i]), protected=bool(ap[i]), token_id=T + i)
        out[p + "app_keys"] = ak
        out[p + "app_radii"] = ar
        out[p + "app_angles"] = aang
        out[p + "app_values"] = av
        out[p + "app_lh"] = np.stack([al, ah], axis=1)
        out[p + "app_tier"] = at.astype(np.int64)
        out[p + "app_prot"] = ap
        _dump_store(p + "app_", st, out)
    np.savez_compressed(os.path.join(OUT, "golden_store.npz"), **out)


def gen_rdr():
    rng = np.random.default_rng(77)
    out = {}
    cases = []
    for ci in range(6):
        L, H, T, d = [(1, 1, 40, 8), (2, 3, 200, 16), (2, 2, 500, 64),
                      (1, 4, 257, 128), (3, 2, 100, 8), (1, 1, 64, 64)][ci]
        tiers = PANEL if d >= 64 else ((0, 0, 0, 0), (1, 2, 2, 0), (2, 4, 4, 0), (3, 8, 8, 0))
        eps = {t[0]: (float(rng.uniform(0.001, 0.3)) / (k + 1), float(rng.uniform(0.001, 0.2)) / (k + 1))
               for k, t in enumerate(tiers[1:])}
        radii = rng.uniform(0.2, 3.0, size=(L, H, T))
        if ci == 4:
            radii[:] = 1.0            # forced nu ties -> flat-index tie order
        if ci == 5:
            radii[:, :, ::2] = 0.0    # zero-radius states (nu tie blocks, +-0)
        seg = rng.integers(0, 3, size=T).astype(np.int8)
        u_hat = rng.uniform(0.2, 1.0, (L, H))
        s_hat = rng.uniform(0.0, 0.8, (L, H))
        r_q = float(rng.uniform(1.0, 40.0))
        omega = np.array([0.02, 2.0, 1.0])
        lam = [0.0, 1e-4, 3e-5, 1e-3, 0.0, 3e-5][ci]
        prot = rng.random((L, H, T)) < [0.0, 0.05, 0.01, 0.0, 0.1, 0.0][ci]
        feat = ControllerFeatures(u_hat=u_hat, s_hat=s_hat, r_q=r_q, omega=omega,
                                  alpha_theta=1.0, alpha_r=1.0, segments=seg, prefill=T)
        tt = table(tiers, eps)
        sc = score_states(radii, feat, tt, lam, prot, d)
        max_rate = codec.rate_bits(tt.max_tier, d)
        full = sum(codec.rate_bits(tt.spec_for(int(x)), d) for x in
                   full_best_tier_assignment(sc, prot, tt).tier.ravel())
        p = f"c{ci}_"
        out[p + "dims"] = np.array([L, H, T, d], dtype=np.int64)
        out[p + "tiers"] = np.array(tiers, dtype=np.int64)
        out[p + "eps"] = np.array([eps[t[0]] for t in tiers[1:]])
        out[p + "radii"] = radii
        out[p + "seg"] = seg
        out[p + "u_hat"] = u_hat
        out[p + "s_hat"] = s_hat
        out[p + "scalars"] = np.array([r_q, lam, 1.0, 1.0])
        out[p + "omega"] = omega
        out[p + "prot"] = prot
        out[p + "best_tier"] = sc.best_tier
        out[p + "score"] = sc.score
        out[p + "nu"] = sc.nu
        out[p + "d_drop"] = sc.d_drop
        budgets = []
        for frac in (0.0, 0.1, 0.3217, 0.7, 1.5):
            b = int(frac * full) if frac < 1.5 else 10 ** 12
            b = max(b, int(np.sum(prot)) * max_rate)
            budgets.append(b)
            g = allocate_greedy(sc, prot, b, tt, d)
            out[p + f"greedy_{len(budgets) - 1}_tier"] = g.tier
            start = full_best_tier_assignment(sc, prot, tt)
            try:
                dt = downtier_before_drop(start, sc, b, tt, d)
                out[p + f"down_{len(budgets) - 1}_tier"] = dt.tier
            except Exception:
                out[p + f"down_{len(budgets) - 1}_tier"] = np.full((L, H, T), -1, np.int16)
        out[p + "budgets"] = np.array(budgets, dtype=np.int64)
        # scalar append scoring on a handful of states
        sel = rng.integers(0, L * H * T, 16)
        rows = []
        for f in sel:
            l, h, i = np.unravel_index(f, (L, H, T))
            key = SphericalKey(float(radii[l, h, i]), np.zeros(d - 1))
            tid, s, nu = score_and_best_tier(StateId(int(l), int(h), int(i)), key, feat, tt,
                                             lam, protected=bool(prot[l, h, i]))
            rows.append([f, tid, s, nu])
        out[p + "scalar"] = np.array(rows, dtype=np.float64)
    np.savez_compressed(os.path.join(OUT, "golden_rdr.npz"), **out)


if __name__ == "__main__":
    gen_codec()
    gen_bitpack()
    gen_store_attend()
    gen_rdr()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
