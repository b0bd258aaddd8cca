"""Pin the CPU oracle (oracle/sphkv_oracle.py) to golden vectors produced by
the real reference (tests/golden/make_golden.py).  Bit-exact for codes,
streams, pages, SPHKV1 bytes and RDR decisions; 1e-12 for fp64 attend."""

import numpy as np
import pytest

from oracle import sphkv_oracle as O


def tiers_of(arr):
    return [tuple(int(x) for x in row) for row in arr]


@pytest.mark.parametrize("d", [2, 3, 8, 64, 128])
def test_encode_and_quantize_bit_exact(golden, d):
    g = golden("codec")
    r, ang = O.encode_batch(g[f"d{d}_keys"])
    assert np.array_equal(r.view(np.uint64), g[f"d{d}_radii"].view(np.uint64))
    assert np.array_equal(ang.view(np.uint64), g[f"d{d}_angles"].view(np.uint64))
    for b in (1, 2, 4, 6, 7, 8, 12, 15, 16):
        codes = O.quantize_angles(ang, b)
        assert np.array_equal(codes.astype(np.uint16), g[f"d{d}_codes_b{b}"]), b
    deq = O.dequantize_angles(g[f"d{d}_codes_b4"].astype(np.uint64), 4)
    assert np.array_equal(deq, g[f"d{d}_deq_b4"])
    assert np.allclose(O.angular_features(deq), g[f"d{d}_feat_b4"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("d", [8, 128])
def test_append_radius_quantizer(golden, d):
    g = golden("codec")
    r = g[f"d{d}_radii"]
    rows = []
    for s in g[f"d{d}_rscales"]:
        for br in (4, 8, 14):
            rows.append([O.append_radius_code(float(x), float(s), br) for x in r])
    assert np.array_equal(np.array(rows), g[f"d{d}_rcodes_append"])


def test_bitpack_streams(golden):
    g = golden("bitpack")
    for bits in list(range(1, 17)) + [20, 31, 53]:
        codes, stream = g[f"b{bits}_codes"], g[f"b{bits}_stream"]
        assert np.array_equal(O.pack_bits(codes, bits), stream)
        assert np.array_equal(O.unpack_bits(stream, bits, codes.size), codes)


def rebuild(g, name):
    p = name + "_"
    L, H, T, d, dv, P, G = (int(x) for x in g[p + "dims"])
    tiers = tiers_of(g[p + "tiers"])
    st = O.pack_pages(tiers, g[p + "z"], g[p + "tier"], g[p + "protected"],
                      g[p + "radii"], g[p + "angles"], g[p + "values"], P)
    return st, (L, H, T, d, dv, P, G), tiers


def check_store(st, g, prefix):
    assert len(st.pages) == int(g[prefix + "n_pages"])
    meta = np.array([[p.tier[0], p.layer, p.head, p.count] for p in st.pages]).reshape(-1, 4)
    assert np.array_equal(meta, g[prefix + "meta"])
    assert np.array_equal(np.array([p.scale for p in st.pages]), g[prefix + "scales"])
    a = [p.angle_stream() for p in st.pages]
    r = [p.radius_stream() for p in st.pages]
    assert [len(x) for x in a] == list(g[prefix + "astream_len"])
    assert np.array_equal(np.concatenate(a) if a else np.zeros(0, np.uint8), g[prefix + "astream"])
    assert np.array_equal(np.concatenate(r) if r else np.zeros(0, np.uint8), g[prefix + "rstream"])
    br = st.resident_breakdown()
    assert [br[k] for k in ("payload", "header", "ptr", "tag", "prot", "frag", "total")] \
        == list(g[prefix + "resident"])
    sb = [st.expected_stream_bytes(l, h) for l in range(st.layers) for h in range(st.heads)]
    assert sb == list(g[prefix + "stream_bytes"])
    blob = np.frombuffer(st.to_bytes(), dtype=np.uint8)
    assert np.array_equal(blob, g[prefix + "sphkv1"])
    # SPHKV1 identity: file size == resident total - frag (store.py:363)
    assert blob.size == br["total"] - br["frag"]


@pytest.mark.parametrize("name", ["small", "panel64", "panel128", "odd"])
def test_pack_pages_and_snapshot_bit_exact(golden, name):
    g = golden("store")
    st, *_ = rebuild(g, name)
    check_store(st, g, name + "_pack_")


@pytest.mark.parametrize("name", ["small", "panel64", "panel128", "odd"])
def test_appends_bit_exact(golden, name):
    g = golden("store")
    st, (L, H, T, d, dv, P, G), _ = rebuild(g, name)
    p = name + "_"
    for i in range(g[p + "app_radii"].size):
        l, h = (int(x) for x in g[p + "app_lh"][i])
        st.append_item(l, h, float(g[p + "app_radii"][i]), g[p + "app_angles"][i],
                       g[p + "app_values"][i], int(g[p + "app_tier"][i]),
                       protected=bool(g[p + "app_prot"][i]), token_id=T + i)
    check_store(st, g, p + "app_")


@pytest.mark.parametrize("name", ["small", "panel64", "panel128", "odd"])
def test_angle_attend_matches_reference(golden, name):
    g = golden("store")
    st, (L, H, T, d, dv, P, G), _ = rebuild(g, name)
    p = name + "_"
    q = g[p + "q"]
    lens = g[p + "logits_len"]
    off = 0
    k = 0
    cache = O.FeatureCache()
    for l in range(L):
        for h in range(H):
            rq, qf = O.query_features(q[l, h])
            for gi in range(G):
                lg, out = O.head_attend(st, l, h, rq[gi], qf[gi], cache)
                want = g[p + "logits"][off: off + lens[k]]
                assert lg.shape == want.shape
                assert np.allclose(lg, want, rtol=1e-12, atol=1e-12)
                assert np.allclose(out, g[p + "outputs"][k], rtol=1e-11, atol=1e-12)
                off += lens[k]
                k += 1


@pytest.mark.parametrize("ci", range(6))
def test_rdr_bit_exact(golden, ci):
    g = golden("rdr")
    p = f"c{ci}_"
    L, H, T, d = (int(x) for x in g[p + "dims"])
    tiers = tiers_of(g[p + "tiers"])
    eps = {t[0]: tuple(g[p + "eps"][k]) for k, t in enumerate(tiers[1:])}
    r_q, lam, at, ar = g[p + "scalars"]
    sc = O.score_states(g[p + "radii"], g[p + "u_hat"], g[p + "s_hat"], r_q, g[p + "omega"],
                        g[p + "seg"], at, ar, tiers, eps, lam, g[p + "prot"], d)
    assert np.array_equal(sc["best_tier"], g[p + "best_tier"])
    for key in ("score", "nu", "d_drop"):
        assert np.array_equal(sc[key].view(np.uint64), g[p + key].view(np.uint64)), key
    for bi, b in enumerate(g[p + "budgets"]):
        z, tier = O.allocate_greedy(sc["best_tier"], sc["nu"], g[p + "prot"], int(b), tiers, d)
        assert np.array_equal(tier, g[p + f"greedy_{bi}_tier"])
        z0, t0 = O.full_best_tier(sc["best_tier"], g[p + "prot"], tiers)
        want = g[p + f"down_{bi}_tier"]
        if np.all(want == -1):
            with pytest.raises(O.Infeasible):
                O.downtier_before_drop(z0, t0, sc["nu"], g[p + "prot"], int(b), tiers, d)
        else:
            _, tier = O.downtier_before_drop(z0, t0, sc["nu"], g[p + "prot"], int(b), tiers, d)
            assert np.array_equal(tier, want)
    om = g[p + "omega"][g[p + "seg"]]
    for f, tid, s, nu in g[p + "scalar"]:
        l, h, i = np.unravel_index(int(f), (L, H, T))
        got = O.score_one(float(g[p + "radii"][l, h, i]), float(g[p + "u_hat"][l, h]),
                          float(g[p + "s_hat"][l, h]), r_q, float(om[i]), at, ar, tiers, eps,
                          lam, d, protected=bool(g[p + "prot"][l, h, i]))
        assert got[0] == int(tid) and got[1] == s and got[2] == nu


def test_lse_merge_matches_full_softmax():
    rng = np.random.default_rng(0)
    logits = rng.standard_normal(100) * 3
    vals = rng.standard_normal((100, 5))
    _, want = O.dense_attend(np.zeros(1), np.zeros((0, 1)), vals[:0])  # empty -> zeros
    assert np.all(want == 0)
    cuts = [0, 10, 10, 55, 100]  # includes an empty split
    m, l, a = [], [], []
    for s, e in zip(cuts[:-1], cuts[1:]):
        seg = logits[s:e]
        if seg.size == 0:
            m.append(-np.inf); l.append(0.0); a.append(np.zeros(5))
            continue
        mm = seg.max()
        w = np.exp(seg - mm)
        m.append(mm); l.append(w.sum()); a.append(w @ vals[s:e])
    out = O.lse_merge(np.array(m), np.array(l), np.array(a))
    w = np.exp(logits - logits.max())
    assert np.allclose(out, (w / w.sum()) @ vals, atol=1e-13)
    assert np.all(O.lse_merge(np.full(3, -np.inf), np.zeros(3), np.zeros((3, 5))) == 0)
