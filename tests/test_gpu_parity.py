"""GPU parity: CUDA path (through the C ABI) vs the reference's golden vectors
and the CPU oracle on identical inputs.

Bit-exact: radii, angle/radius codes, page streams, SPHKV1 bytes, appends,
RDR best tier / score / nu / allocations.  Tolerance (north_star): logits
max |dl| / max(1, |l|) <= 1e-3 and outputs ||do||_inf / ||o||_inf <= 1e-3.
"""

import math

import numpy as np
import pytest

from oracle import sphkv_oracle as O

pytestmark = pytest.mark.gpu

LOGIT_TOL = 1e-3
OUT_TOL = 1e-3


@pytest.fixture(scope="module")
def sk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_18856_b200 as sk
    from paper_2605_18856_b200 import _lib

    _lib.require_gpu()
    return sk


def table(sk, rows, eps=None):
    t = sk.TierTable(tuple(sk.TierSpec(*map(int, r)) for r in rows))
    for k, s in enumerate(t.non_drop):
        e = eps[k] if eps is not None else (0.01 / (k + 1), 0.005 / (k + 1))
        t.eps_theta[s.id], t.eps_r[s.id] = float(e[0]), float(e[1])
    return t


def boundary_distance(angle, bits, polar):
    step = O.polar_step(bits) if polar else O.circular_step(bits)
    x = angle / step
    return abs(x - math.floor(x) - 0.5)


# ---------------------------------------------------------------------------
# encoder / quantizer
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("d", [2, 3, 8, 64, 128])
def test_encoder_matches_golden(sk, golden, d):
    g = golden("codec")
    r, ang = sk.encode_batch(g[f"d{d}_keys"])
    assert np.array_equal(r.view(np.uint64), g[f"d{d}_radii"].view(np.uint64)), "radii bits"
    want = g[f"d{d}_angles"]
    ulp = np.abs(ang - want) / np.maximum(np.spacing(np.abs(want)), 1e-300)
    assert np.all((ang == want) | (ulp <= 4)), f"max ulp {ulp.max()}"
    flips = 0
    for b in (1, 2, 4, 6, 7, 8, 12, 15, 16):
        codes = sk.quantize_angles(ang, b).astype(np.uint16)
        bad = np.argwhere(codes != g[f"d{d}_codes_b{b}"])
        for i, j in bad:  # a flip is only legal on a rounding boundary (libm ulp tie)
            assert boundary_distance(want[i, j], b, j < d - 2) < 1e-9, (b, i, j)
        flips += len(bad)
    assert flips <= 2


@pytest.mark.parametrize("d", [2, 8, 64, 128])
def test_quantizer_bit_exact_on_reference_angles(sk, golden, d):
    g = golden("codec")
    for b in (1, 2, 4, 6, 7, 8, 12, 15, 16):
        codes = sk.quantize_angles(g[f"d{d}_angles"], b).astype(np.uint16)
        assert np.array_equal(codes, g[f"d{d}_codes_b{b}"]), b


def test_angles_from_unit_and_zero_vector(sk):
    s = sk.to_spherical(np.zeros(4))
    assert s.radius == 0.0 and np.all(s.angles == 0.0)
    s = sk.to_spherical(np.array([0.0, 2.0]))
    assert s.radius == pytest.approx(2.0) and s.angles == pytest.approx([math.pi / 2])
    u = np.random.default_rng(0).standard_normal((50, 9))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    assert np.allclose(sk.angles_from_unit(u), O.angles_from_unit(u), rtol=0, atol=1e-14)


# ---------------------------------------------------------------------------
# packer / export / appends
# ---------------------------------------------------------------------------

CASES = ["small", "panel64", "panel128", "odd"]


def pack_case(sk, g, name, from_keys=False):
    p = name + "_"
    L, H, T, d, dv, P, G = (int(x) for x in g[p + "dims"])
    tiers = table(sk, g[p + "tiers"])
    asg = sk.TierAssignment(g[p + "z"], g[p + "tier"], g[p + "protected"])
    if P % 32:
        pytest.skip("device pages are multiples of 32 items")
    if not from_keys:
        st = sk.pack_pages_arrays(asg, g[p + "radii"], g[p + "angles"], g[p + "values"], tiers, P)
    else:
        st = sk.PagedStore(tiers, L, H, d, dv, P, capacity_tokens=T)
        sk.pack_device(st, keys=g[p + "keys"].reshape(-1, d), radii=g[p + "radii"].reshape(-1),
                       values=g[p + "values"].reshape(-1, dv), z=g[p + "z"].reshape(-1),
                       tier=g[p + "tier"].reshape(-1), protect=g[p + "protected"].reshape(-1),
                       tokens=T)
    return st, tiers, (L, H, T, d, dv, P, G)


def check_store_bytes(st, g, prefix):
    pages = st.pages
    assert len(pages) == int(g[prefix + "n_pages"])
    meta = np.array([[p.tier.id, p.layer, p.head, p.count] for p in pages]).reshape(-1, 4)
    assert np.array_equal(meta, g[prefix + "meta"])
    assert np.array_equal(np.array([p.radius_scale for p in pages]), g[prefix + "scales"])
    a = [p.angle_stream() for p in pages]
    assert np.array_equal(np.concatenate(a) if a else np.zeros(0, np.uint8), g[prefix + "astream"])
    r = [p.radius_stream() for p in pages]
    assert np.array_equal(np.concatenate(r) if r else np.zeros(0, np.uint8), g[prefix + "rstream"])
    br = st.resident_breakdown()
    assert [br.payload_bytes, br.header_bytes, br.ptr_bytes, br.tag_bytes, br.prot_bytes,
            br.frag_bytes, br.total] == list(g[prefix + "resident"])
    blob = np.frombuffer(st.to_bytes(), dtype=np.uint8)
    assert np.array_equal(blob, g[prefix + "sphkv1"])
    assert blob.size == br.total - br.frag_bytes
    st.check_invariants()


@pytest.mark.parametrize("name", CASES)
def test_pack_pages_bit_exact(sk, golden, name):
    g = golden("store")
    st, *_ = pack_case(sk, g, name)
    check_store_bytes(st, g, name + "_pack_")
    # the device block (word-interleaved item-major layout, sphkv_b200.h)
    # holds exactly the reference codes: decode it on the host and compare
    # with the reference SoA stream (store.py:205-208)
    P, d = st.page_size, st.d
    for p in st.pages:
        if p.count == 0:
            continue
        row = st._host()[1][p.index]
        b = int(row["abits"])
        W = (((d - 1) * b + 31) // 32 + 3) // 4 * 4
        nw = (P + 31) // 32 * W * 32
        off = int(row["code_off"])
        words = st.t_codes[off: off + 4 * nw].cpu().numpy().view(np.uint32)
        i = np.arange(p.count)[:, None]
        w = np.arange(W)[None, :]
        idx = (((i >> 5) * (W >> 2) + (w >> 2)) * 32 + (i & 31)) * 4 + (w & 3)
        strings = words[idx].astype(np.uint64)  # [count, W]
        bits = ((strings[:, :, None] >> np.arange(32, dtype=np.uint64)) & 1).reshape(p.count, -1)
        j = np.arange(d - 1)
        codes = np.zeros((p.count, d - 1), dtype=np.uint64)
        for t in range(b):
            codes |= bits[:, j * b + t] << np.uint64(t)
        want = O.unpack_bits(p.angle_stream(), b, p.count * (d - 1)).reshape(d - 1, p.count).T
        assert np.array_equal(codes, want.astype(np.uint64))


@pytest.mark.parametrize("name", CASES)
def test_pack_from_dense_keys(sk, golden, name):
    g = golden("store")
    st, *_ = pack_case(sk, g, name, from_keys=True)
    check_store_bytes(st, g, name + "_pack_")


@pytest.mark.parametrize("name", CASES)
def test_appends_bit_exact(sk, golden, name):
    g = golden("store")
    st, tiers, (L, H, T, d, dv, P, G) = pack_case(sk, g, name)
    p = name + "_"
    for i in range(g[p + "app_radii"].size):
        l, h = (int(x) for x in g[p + "app_lh"][i])
        key = sk.SphericalKey(float(g[p + "app_radii"][i]), g[p + "app_angles"][i])
        st.append_item(l, h, key, g[p + "app_values"][i], int(g[p + "app_tier"][i]),
                       protected=bool(g[p + "app_prot"][i]), token_id=T + i)
    check_store_bytes(st, g, p + "app_")


@pytest.mark.parametrize("stage", ["pack", "app"])
@pytest.mark.parametrize("name", CASES)
def test_sphkv1_import_roundtrip(sk, golden, name, stage, tmp_path):
    """SPHKV1 import into device pages (store.py:391-427; reference
    test_store.py:284-305): the reference's own snapshot bytes load, export
    back byte-identical, keep the size + frag == resident identity, and the
    loaded pages attend exactly like the packed ones."""
    g = golden("store")
    p = name + "_"
    L, H, T, d, dv, P, G = (int(x) for x in g[p + "dims"])
    if P % 32:
        pytest.skip("device pages are multiples of 32 items")
    tiers = table(sk, g[p + "tiers"])
    blob = g[p + stage + "_sphkv1"].tobytes()
    path = tmp_path / "snap.bin"
    path.write_bytes(blob)
    st = sk.PagedStore.from_file(str(path), tiers)
    br = st.resident_breakdown()
    assert st.to_bytes() == blob
    assert len(blob) + br.frag_bytes == br.total == int(g[p + stage + "_resident"][-1])
    st.check_invariants()
    assert all(np.all(pg.token_ids == -1) for pg in st.pages)
    ref, *_ = pack_case(sk, g, name)
    for l in range(L):
        for h in range(H):
            a_lg, a_out = sk.decode.attend_heads(ref, l, h, g[p + "q"][l, h])
            b_lg, b_out = sk.decode.attend_heads(st, l, h, g[p + "q"][l, h])
            if stage == "pack":
                assert np.array_equal(a_lg, b_lg) and np.array_equal(a_out, b_out)
    # appends keep working on an imported store (pools, pointer lists, group_last)
    st.append_item(0, 0, sk.SphericalKey(0.5, np.full(d - 1, 0.3)), np.ones(dv),
                   int(tiers.non_drop[0].id))
    st.check_invariants()
    with pytest.raises(ValueError):
        sk.PagedStore.from_bytes(b"NOTSPH" + blob[6:], tiers)


# ---------------------------------------------------------------------------
# attend
# ---------------------------------------------------------------------------

def assert_attend_close(lg, out, want_lg, want_out):
    assert lg.shape == want_lg.shape
    if want_lg.size:
        err = np.max(np.abs(lg - want_lg) / np.maximum(1.0, np.abs(want_lg)))
        assert err <= LOGIT_TOL, err
    den = max(np.max(np.abs(want_out)), 1e-30)
    assert np.max(np.abs(out - want_out)) / den <= OUT_TOL


@pytest.mark.parametrize("name", CASES)
def test_ada_attend_matches_reference_golden(sk, golden, name):
    g = golden("store")
    st, tiers, (L, H, T, d, dv, P, G) = pack_case(sk, g, name)
    p = name + "_"
    lens = g[p + "logits_len"]
    off = k = 0
    for l in range(L):
        for h in range(H):
            lg, out = sk.decode.attend_heads(st, l, h, g[p + "q"][l, h])
            for gi in range(G):
                want = g[p + "logits"][off: off + lens[k]]
                assert_attend_close(lg[gi], out[gi], want, g[p + "outputs"][k])
                off += lens[k]
                k += 1


def test_empty_head_yields_zero_output(sk):
    tiers = table(sk, [(0, 0, 0, 0), (1, 4, 6, 0)])
    L, H, T, d = 1, 2, 64, 8
    rng = np.random.default_rng(0)
    keys = rng.standard_normal((L, H, T, d))
    r, a = O.encode_batch(keys.reshape(-1, d))
    z = np.ones((L, H, T), np.int8)
    z[0, 1] = 0
    tier = z.astype(np.int16)
    asg = sk.TierAssignment(z, tier, np.zeros((L, H, T), bool))
    st = sk.pack_pages_arrays(asg, r.reshape(L, H, T), a.reshape(L, H, T, d - 1),
                              rng.standard_normal((L, H, T, d)), tiers, 32)
    lg, out = sk.decode.attend_heads(st, 0, 1, rng.standard_normal((3, d)))
    assert lg.shape == (3, 0) and np.all(out == 0)
    assert sk.angle_logits(np.ones(d), st, 0, 1).size == 0


def test_split_merge_equals_single_pass(sk):
    """Many page-range splits merged by the LSE kernel == one softmax (decode.py:347-354)."""
    import torch

    wl = sk.synth.generate(1, 1, 2, 4, 4096, 64, seed=3)
    tiers = table(sk, [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)])
    st = sk.PagedStore(tiers, 1, 2, 64, 64, 128, capacity_tokens=4096)
    n = wl.groups * wl.tokens
    rng = np.random.default_rng(1)
    tier = rng.choice([0, 1, 2, 3], n, p=[0.1, 0.4, 0.4, 0.1]).astype(np.int16)
    radii = torch.empty(n, dtype=torch.float64, device="cuda")
    from paper_2605_18856_b200 import _lib
    _lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, 64,
                                             radii.data_ptr(), _lib.stream_ptr()))
    sk.pack_device(st, keys=wl.keys.view(-1, 64), radii=radii, values=wl.values.view(-1, 64),
                   z=(tier != 0).astype(np.int8), tier=tier, protect=np.zeros(n, np.uint8),
                   tokens=wl.tokens)
    one = sk.ada_decode(st, wl.queries, sk.plan_store(st, grid=2, units_per_cta=1))
    many = sk.ada_decode(st, wl.queries, sk.plan_store(st, grid=148, units_per_cta=4))
    assert torch.allclose(one, many, rtol=2e-5, atol=2e-5)
    # repeated fused launches reuse the self re-arming split counters
    plan = sk.plan_store(st, grid=148, units_per_cta=1)
    for _ in range(3):
        again = sk.ada_decode(st, wl.queries, plan)
        assert torch.allclose(one, again, rtol=2e-5, atol=2e-5)
    assert int(plan.ctl.abs().sum()) == 0


def _mixed_store(sk, T, G=4, d=64, H=2, seed=3, P=128):
    import torch
    from paper_2605_18856_b200 import _lib

    wl = sk.synth.generate(1, 1, H, G, T, d, seed=seed)
    tiers = table(sk, [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)])
    st = sk.PagedStore(tiers, 1, H, d, d, P, capacity_tokens=T)
    n = wl.groups * wl.tokens
    rng = np.random.default_rng(seed)
    tier = rng.choice([0, 1, 2, 3], n, p=[0.1, 0.4, 0.4, 0.1]).astype(np.int16)
    radii = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, d,
                                             radii.data_ptr(), _lib.stream_ptr()))
    sk.pack_device(st, keys=wl.keys.view(-1, d), radii=radii, values=wl.values.view(-1, d),
                   z=(tier != 0).astype(np.int8), tier=tier, protect=np.zeros(n, np.uint8),
                   tokens=wl.tokens)
    return st, wl


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("G", [1, 3, 4])
def test_two_bit_hbyte_tables_with_deaths(sk, d, G):
    """2-bit tier through the per-query h-byte tables (G <= 4): matches the
    oracle's recurrence, including items whose codes hit 0 or 3 (sine 0 ->
    every later feature is 0): early deaths send the tile to the exact
    generic path, late deaths are masked per item."""
    rng = np.random.default_rng(d + G)
    L, H, T, P = 1, 2, 1500, 256
    tl = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8)]
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    keys = rng.standard_normal((L, H, T, d))
    # deaths: a key along an axis has polar angle 0 there (code 0); a key whose
    # tail vanishes after coordinate j has angle 0/pi at j (code 0 or 3)
    keys[0, 0, 10, :] = 0.0
    keys[0, 0, 10, 7] = 2.0                       # early death (row 7), tile 0
    keys[0, 1, 700:705, d - 20:] = 0.0             # late deaths (rows ~d-21)
    keys[0, 1, 900, d - 6:] = 0.0
    keys[0, 1, 901, :] = -keys[0, 1, 901, :] * 0 + np.eye(d)[d - 3] * -1.5
    r, ang = O.encode_batch(keys.reshape(-1, d))
    r, ang = r.reshape(L, H, T), ang.reshape(L, H, T, d - 1)
    tier = np.where(rng.random((L, H, T)) < 0.85, 1, 2).astype(np.int16)
    z = np.ones((L, H, T), np.int8)
    prot = np.zeros((L, H, T), bool)
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    st = sk.pack_pages_arrays(sk.TierAssignment(z, tier, prot), r, ang, vals, tiers, P)
    assert not st.uses_hb(G)  # opt-in
    st.hbyte_tables = True
    assert st.uses_hb(G)
    ost = O.pack_pages(tl, z, tier, prot, r, ang, vals, P)
    for h in range(H):
        q = rng.standard_normal((G, d)) * 4
        lg, out = sk.decode.attend_heads(st, 0, h, q)
        rq, qf = O.query_features(q)
        for g in range(G):
            want_lg, want_out = O.head_attend(ost, 0, h, rq[g], qf[g])
            assert_attend_close(lg[g], out[g], want_lg, want_out)
        # the fused launch (h-byte tables built per unit) gives the same outputs
        import torch

        qd = torch.zeros((st.groups, G, d), dtype=torch.float32, device="cuda")
        qd[st._group(0, h)] = torch.as_tensor(q, dtype=torch.float32, device="cuda")
        fused = sk.ada_decode(st, qd, sk.plan_store(st, groups=[st._group(0, h)], grid=3,
                                                   units_per_cta=1))
        assert np.max(np.abs(fused.double().cpu().numpy() - out)) <= 1e-5 * max(1, np.abs(out).max())


def test_unit_longer_than_tile_cap(sk, monkeypatch):
    """A unit with more tiles than the kernel's tile list holds (a direct C-ABI
    caller's plan) runs as several segments with one online softmax: same
    outputs as a planner-split plan, logits included."""
    import torch
    from paper_2605_18856_b200 import plan as planmod

    st, wl = _mixed_store(sk, 150000)
    ref = sk.ada_decode(st, wl.queries, sk.plan_store(st, grid=148, units_per_cta=1))
    cap = planmod.tile_geometry()
    monkeypatch.setattr(planmod, "tile_geometry", lambda: (cap[0], 1 << 20))
    big = sk.plan_store(st, groups=[0], grid=1, units_per_cta=1)
    assert big.n_units == 1 and int(big.group_items[0]) > 2 * 512 * cap[0]
    # the standard fused kernel flags the unit (error word) instead of truncating it
    big.check_units = True
    with pytest.raises(RuntimeError):
        sk.ada_decode(st, wl.queries, big)
    assert int(big.ctl.abs().sum()) == 0
    # the general kernel runs it as segments (gate margins / debug logits paths)
    m = torch.empty(4, dtype=torch.float32, device="cuda")
    got = sk.ada_decode(st, wl.queries, big, margins=m)
    assert torch.allclose(ref[:4], got, rtol=2e-5, atol=2e-5)
    lg = torch.zeros(int(big.group_items.sum()) * 4, dtype=torch.float32, device="cuda")
    got2 = sk.ada_decode(st, wl.queries, big, logits=lg)
    assert torch.allclose(ref[:4], got2, rtol=2e-5, atol=2e-5)
    monkeypatch.undo()
    want_lg, _ = sk.decode.attend_heads(st, 0, 0, wl.queries[0].double().cpu().numpy())
    n0 = int(big.group_items[0])
    assert np.allclose(lg[: n0 * 4].view(n0, 4).T.double().cpu().numpy(), want_lg, rtol=1e-5,
                       atol=1e-5)


def test_dynamic_plan_back_to_back(sk):
    """Dynamic-queue plans launched back to back on one stream (programmatic
    dependent launch): no CTA claims from the queue before the previous grid
    is done, so every launch equals the static plan and the control words
    end re-armed."""
    import torch

    st, wl = _mixed_store(sk, 60000, seed=4)
    ref = sk.ada_decode(st, wl.queries, sk.plan_store(st, grid=148, units_per_cta=1))
    dyn = sk.plan_store(st, grid=40, units_per_cta=4, dynamic=True)
    outs = [torch.empty_like(ref) for _ in range(6)]
    for o in outs:
        sk.ada_decode(st, wl.queries, dyn, out=o)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.allclose(ref, o, rtol=2e-5, atol=2e-5)
    assert int(dyn.ctl.abs().sum()) == 0


@pytest.mark.parametrize("kw", [dict(grid=148, units_per_cta=1),
                                dict(grid=40, units_per_cta=1, tail=0.3, tail_pieces=3),
                                dict(grid=40, units_per_cta=4, dynamic=True)])
def test_pipelined_unit_transitions_match_standard(sk, kw, monkeypatch):
    """k_ada_decode_pipe (SPHKV_PIPE=1: one continuous tile sequence across a
    CTA's units, merges deferred to the CTA's end) gives the standard kernel
    body's outputs bit for bit, back to back under PDL, and re-arms every
    control word."""
    import torch

    st, wl = _mixed_store(sk, 60000, seed=6)
    plan = sk.plan_store(st, **kw)
    monkeypatch.setenv("SPHKV_PIPE", "0")
    ref = sk.ada_decode(st, wl.queries, plan)
    torch.cuda.synchronize()
    monkeypatch.setenv("SPHKV_PIPE", "1")
    outs = [torch.empty_like(ref) for _ in range(4)]
    for o in outs:
        sk.ada_decode(st, wl.queries, plan, out=o)
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(ref, o)
    assert int(plan.ctl.abs().sum()) == 0


@pytest.mark.parametrize("world", [2, 3, 8])
def test_page_range_split_two_level_merge(sk, world):
    """Multi-GPU data path on one device: each simulated rank decodes its
    page range (plan_store_range), merges its splits to one state per
    (group, q-head) (lse_merge_ex state_out=1), the states are laid out rank-
    major as all_gather_into_tensor produces them, and merge_gathered must
    equal the single-pass decode."""
    import torch
    from paper_2605_18856_b200 import _lib, plan as planmod

    wl = sk.synth.generate(1, 2, 2, 4, 3000, 64, seed=5)
    tiers = table(sk, [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)])
    st = sk.PagedStore(tiers, 2, 2, 64, 64, 128, capacity_tokens=3000)
    n = wl.groups * wl.tokens
    rng = np.random.default_rng(2)
    tier = rng.choice([0, 1, 2, 3], n, p=[0.1, 0.4, 0.4, 0.1]).astype(np.int16)
    radii = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, 64,
                                             radii.data_ptr(), _lib.stream_ptr()))
    sk.pack_device(st, keys=wl.keys.view(-1, 64), radii=radii, values=wl.values.view(-1, 64),
                   z=(tier != 0).astype(np.int8), tier=tier, protect=np.zeros(n, np.uint8),
                   tokens=wl.tokens)
    groups = list(range(wl.groups))
    want = sk.ada_decode(st, wl.queries, sk.plan_store(st, groups=groups))
    G, dv = 4, 64
    F = G * (dv + 2)
    gathered = torch.empty((world, len(groups), F), dtype=torch.float32, device="cuda")
    for r in range(world):
        p = planmod.plan_store_range(st, groups, r, world, grid=16)
        parts = sk.decode._partials(p, G, dv)
        _lib.check(_lib.lib().sphkv_ada_decode(st.cptr_for(G), wl.queries.data_ptr(), G,
                                               p.units.data_ptr(), p.n_units, parts.data_ptr(),
                                               None, None, p.grid, _lib.stream_ptr()))
        planmod.merge_local_state(p, parts, G, dv, gathered[r])
        # the fused single-launch form (in-kernel merge emits the rank's state)
        fused = sk.decode.ada_decode_state(st, wl.queries, p)
        assert torch.allclose(fused, gathered[r], rtol=2e-5, atol=2e-5)
        gathered[r] = fused
    out = torch.empty_like(want)
    planmod.merge_gathered(len(groups), world, gathered, G, dv, out)
    assert torch.allclose(out, want, rtol=2e-5, atol=2e-5)


def test_config1_geometry_vs_oracle(sk):
    """1 layer, 8 KV / 32 Q heads, d=128, T=8K, P=256, panel tiers, RDR at a
    ~30% KV-byte reduction: page bytes exact, attend within tolerance."""
    import torch
    from paper_2605_18856_b200 import synth

    H, G, T, d = 8, 4, 8192, 128
    wl = synth.generate(1, 1, H, G, T, d, seed=0)
    keys64 = wl.keys.double().cpu().numpy().reshape(-1, d)
    r, ang = O.encode_batch(keys64)
    eps = {1: (0.2, 0.03), 2: (0.06, 0.008), 3: (0.015, 0.002), 4: (0.008, 0.002),
           5: (0.0005, 0.00005), 6: (0.00006, 0.00001)}
    tiers = synth.panel_tiers(eps=eps)
    tl = [(t.id, t.angle_bits, t.radius_bits, t.meta_bits) for t in tiers.tiers]
    u_hat, s_hat, r_q = synth.features(wl)
    seg = wl.segments
    omega = np.array(synth.PANEL_OMEGA)
    prot = np.zeros((1, H, T), bool)
    sc = O.score_states(r.reshape(1, H, T), u_hat.reshape(1, H), s_hat.reshape(1, H), r_q, omega,
                        seg, 1.0, 1.0, tl, eps, synth.PANEL_LAMBDA, prot, d)
    dense_bits = H * T * d * 16
    z, tier = O.allocate_greedy(sc["best_tier"], sc["nu"], prot, int(0.3217 * dense_bits), tl, d)
    vals = wl.values.float().cpu().numpy().reshape(1, H, T, d).astype(np.float64)
    ost = O.pack_pages(tl, z, tier, prot, r.reshape(1, H, T), ang.reshape(1, H, T, d - 1),
                       vals, 256)
    st = sk.PagedStore(tiers, 1, H, d, d, 256, capacity_tokens=T)
    sk.pack_device(st, keys=wl.keys.view(-1, d), radii=r, values=wl.values.view(-1, d),
                   z=z.reshape(-1), tier=tier.reshape(-1), protect=prot.reshape(-1), tokens=T)
    assert st.n_pages == len(ost.pages)
    assert np.frombuffer(st.to_bytes(), np.uint8).tobytes() == ost.to_bytes()
    # attend: every (kv head, q head)
    q = wl.queries.double().cpu().numpy()
    lgbuf = torch.zeros(st.retained_count() * G, dtype=torch.float32, device="cuda")
    plan = sk.plan_store(st)
    out = sk.ada_decode(st, wl.queries, plan, logits=lgbuf).double().cpu().numpy()
    lg_all = lgbuf.double().cpu().numpy()
    cache = O.FeatureCache()
    off = 0
    for h in range(H):
        rq, qf = O.query_features(q[h])
        n = int(plan.group_items[h])
        lg = lg_all[off * G: (off + n) * G].reshape(n, G)
        for gi in range(G):
            want_lg, want_out = O.head_attend(ost, 0, h, rq[gi], qf[gi], cache)
            assert_attend_close(lg[:, gi], out[h * G + gi], want_lg, want_out)
        off += n


# ---------------------------------------------------------------------------
# dense baseline
# ---------------------------------------------------------------------------

def test_dense_decode_vs_oracle(sk):
    import torch
    from paper_2605_18856_b200 import synth

    wl = synth.generate(1, 2, 2, 4, 3000, 128, seed=5)
    ds = sk.DenseStore(2, 2, 128, 128, 256)
    ds.bulk_load(wl.keys, wl.values)
    out = sk.dense_decode(ds, wl.queries).double().cpu().numpy()
    keys = wl.keys.double().cpu().numpy()
    vals = wl.values.double().cpu().numpy()
    q = wl.queries.double().cpu().numpy()
    for g in range(wl.groups):
        for gi in range(4):
            _, want = O.dense_attend(q[g, gi], keys[g], vals[g])
            err = np.max(np.abs(out[g * 4 + gi] - want)) / np.max(np.abs(want))
            assert err <= 5e-3, err  # bf16 K / q in the dense baseline


def test_dense_head_attend_reference_shape(sk):
    """_head_attend("dense") (decode.py:302-307) returns every logit (one per
    token, decode.py:63-69 on the stored bf16 keys), the dense output and the
    reference meter counts (store.py:533-546); view() un-swizzles the pages;
    dense_logits runs in fp64 on the device."""
    from paper_2605_18856_b200 import synth

    wl = synth.generate(1, 2, 2, 4, 700, 64, seed=9)
    ds = sk.DenseStore(2, 2, 64, 64, 256)
    ds.bulk_load(wl.keys, wl.values)
    keys = wl.keys.double().cpu().numpy()
    vals = wl.values.double().cpu().numpy()
    q = wl.queries.double().cpu().numpy()[1 * 2 + 1, 2]
    kv, vv = ds.view(1, 1)
    assert np.array_equal(kv, keys[3]) and np.array_equal(vv, vals[3])
    ds.meter.reset()
    lg, out, n, _ = sk.decode._head_attend("dense", ds, 1, 1, q)
    want_lg, want_out = O.dense_attend(q, keys[3], vals[3])
    assert n == 700 and lg.shape == (700,)
    assert np.max(np.abs(lg - want_lg) / np.maximum(1, np.abs(want_lg))) < 1e-5
    assert np.max(np.abs(out - want_out)) / np.max(np.abs(want_out)) < 5e-3  # bf16 q in the kernel
    snap = ds.meter.snapshot()
    assert snap["header"] == 16 * 3 and snap["dense_k_read"] == 700 * 64 * 2
    assert snap["values"] == 700 * 64 * 2
    rng = np.random.default_rng(3)
    kk, qq = rng.standard_normal((333, 48)), rng.standard_normal(48)
    np.testing.assert_allclose(sk.dense_logits(qq, kk), kk @ qq / math.sqrt(48), rtol=1e-13,
                               atol=1e-13)
    with pytest.raises(ValueError):
        sk.dense_logits(qq, kk[:, :40])


def test_angle_head_attend_meters_stream_bytes(sk):
    """_head_attend("angle") meters header + code + value bytes of every
    listed page once per call (decode.py:336-342), = expected_stream_bytes."""
    rng = np.random.default_rng(11)
    L, H, T, d, P = 1, 2, 900, 64, 256
    tl = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)]
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    r, ang = O.encode_batch(rng.standard_normal((L * H * T, d)))
    tier = rng.choice([0, 1, 2, 3], (L, H, T)).astype(np.int16)
    st = sk.pack_pages_arrays(sk.TierAssignment((tier != 0).astype(np.int8), tier,
                                                np.zeros((L, H, T), bool)),
                              r.reshape(L, H, T), ang.reshape(L, H, T, d - 1),
                              rng.standard_normal((L, H, T, d)), tiers, P)
    st.meter.reset()
    sk.decode._head_attend("angle", st, 0, 1, rng.standard_normal(d))
    snap = st.meter.snapshot()
    assert snap["header"] + snap["k_codes"] + snap["values"] == st.expected_stream_bytes(0, 1)
    assert snap["dense_k_read"] == snap["dense_k_write"] == 0


def test_pack_values_single_rounding(sk):
    """Values are rounded to fp16 once, as numpy astype(np.float16) does
    (store.py:383), for float64 host arrays and float64 device tensors."""
    import torch

    rng = np.random.default_rng(2)
    L, H, T, d, P = 1, 1, 2048, 64, 256
    tl = [(0, 0, 0, 0), (1, 4, 8, 8)]
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    r, ang = O.encode_batch(rng.standard_normal((T, d)))
    vals = rng.standard_normal((L, H, T, d))
    asg = sk.TierAssignment(np.ones((L, H, T), np.int8), np.ones((L, H, T), np.int16),
                            np.zeros((L, H, T), bool))
    st = sk.pack_pages_arrays(asg, r.reshape(L, H, T), ang.reshape(L, H, T, d - 1), vals, tiers, P)
    got = np.concatenate([p.values for p in st.pages])
    want = vals.reshape(T, d).astype(np.float16).astype(np.float64)
    assert np.array_equal(got, want)
    out = sk._lib.to_f16(torch.as_tensor(vals.reshape(-1), device="cuda"))
    assert np.array_equal(out.cpu().numpy(), vals.reshape(-1).astype(np.float16))


# ---------------------------------------------------------------------------
# RDR
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("ci", range(6))
def test_rdr_bit_exact(sk, golden, ci):
    g = golden("rdr")
    p = f"c{ci}_"
    L, H, T, d = (int(x) for x in g[p + "dims"])
    tiers = table(sk, g[p + "tiers"], g[p + "eps"])
    r_q, lam, at, ar = g[p + "scalars"]
    feat = sk.ControllerFeatures(u_hat=g[p + "u_hat"], s_hat=g[p + "s_hat"], r_q=float(r_q),
                                 omega=g[p + "omega"], alpha_theta=float(at), alpha_r=float(ar),
                                 segments=g[p + "seg"], prefill=T)
    sc = sk.score_states(g[p + "radii"], feat, tiers, float(lam), g[p + "prot"], d)
    assert np.array_equal(sc.best_tier, g[p + "best_tier"])
    for key in ("score", "nu", "d_drop"):
        assert np.array_equal(getattr(sc, key).view(np.uint64), g[p + key].view(np.uint64)), key
    for bi, b in enumerate(g[p + "budgets"]):
        asg = sk.allocate_greedy(sc, g[p + "prot"], int(b), tiers, d)
        assert np.array_equal(asg.tier, g[p + f"greedy_{bi}_tier"]), ("greedy", bi)
        start = sk.full_best_tier_assignment(sc, g[p + "prot"], tiers)
        want = g[p + f"down_{bi}_tier"]
        if np.all(want == -1):
            with pytest.raises(sk.InfeasibleProtectionError):
                sk.downtier_before_drop(start, sc, int(b), tiers, d)
        else:
            assert np.array_equal(sk.downtier_before_drop(start, sc, int(b), tiers, d).tier, want)


def test_greedy_large_random_vs_oracle(sk):
    """Exact parallel greedy vs the sequential oracle on 200K states with ties."""
    rng = np.random.default_rng(11)
    L, H, T, d = 2, 4, 25000, 128
    tl = [tuple(x) for x in ((0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 6, 8, 8),
                             (4, 7, 8, 8), (5, 12, 14, 8), (6, 15, 16, 8))]
    eps = {k: (0.3 / k ** 2, 0.05 / k ** 2) for k in range(1, 7)}
    tiers = table(sk, tl, [eps[k] for k in range(1, 7)])
    radii = np.round(rng.uniform(0.2, 3.0, (L, H, T)), 2)  # many exact nu ties
    seg = rng.integers(0, 3, T).astype(np.int8)
    u_hat, s_hat = rng.uniform(0.2, 1, (L, H)), rng.uniform(0, 0.8, (L, H))
    prot = rng.random((L, H, T)) < 0.01
    feat = sk.ControllerFeatures(u_hat=u_hat, s_hat=s_hat, r_q=30.0, omega=np.array([0.02, 2, 1.0]),
                                 alpha_theta=1.0, alpha_r=1.0, segments=seg, prefill=T)
    sc = sk.score_states(radii, feat, tiers, 3e-5, prot, d)
    osc = O.score_states(radii, u_hat, s_hat, 30.0, np.array([0.02, 2, 1.0]), seg, 1.0, 1.0, tl,
                         eps, 3e-5, prot, d)
    assert np.array_equal(sc.nu.view(np.uint64), osc["nu"].view(np.uint64))
    full = sum(O.rate_bits(tl[int(t)], d) for t in osc["best_tier"].ravel())
    for frac in (0.05, 0.3217, 0.8):
        b = int(frac * full)
        asg = sk.allocate_greedy(sc, prot, b, tiers, d)
        _, want = O.allocate_greedy(osc["best_tier"], osc["nu"], prot, b, tl, d)
        assert np.array_equal(asg.tier, want), frac
        z0, t0 = O.full_best_tier(osc["best_tier"], prot, tl)
        _, want_d = O.downtier_before_drop(z0, t0, osc["nu"], prot, b, tl, d)
        got_d = sk.downtier_before_drop(sk.full_best_tier_assignment(sc, prot, tiers), sc, b, tiers, d)
        assert np.array_equal(got_d.tier, want_d), frac


def test_scalar_append_scoring_matches_golden(sk, golden):
    g = golden("rdr")
    for ci in range(6):
        p = f"c{ci}_"
        L, H, T, d = (int(x) for x in g[p + "dims"])
        tiers = table(sk, g[p + "tiers"], g[p + "eps"])
        r_q, lam, at, ar = g[p + "scalars"]
        feat = sk.ControllerFeatures(u_hat=g[p + "u_hat"], s_hat=g[p + "s_hat"], r_q=float(r_q),
                                     omega=g[p + "omega"], alpha_theta=float(at),
                                     alpha_r=float(ar), segments=g[p + "seg"], prefill=T)
        for f, tid, s, nu in g[p + "scalar"]:
            l, h, i = np.unravel_index(int(f), (L, H, T))
            key = sk.SphericalKey(float(g[p + "radii"][l, h, i]), np.zeros(d - 1))
            got = sk.score_and_best_tier(sk.StateId(int(l), int(h), int(i)), key, feat, tiers,
                                         float(lam), protected=bool(g[p + "prot"][l, h, i]))
            assert got[0] == int(tid) and got[1] == s and got[2] == nu


@pytest.mark.parametrize("name", ["small", "rows"])
def test_compute_features_matches_reference_golden(sk, golden, name):
    """controller.compute_features (controller.py:99-142) on the device (fp64)
    vs the reference's own outputs on the same workload."""
    from types import SimpleNamespace

    g = golden("features")
    p = name + "_"
    wl = SimpleNamespace(keys=g[p + "keys"], queries=g[p + "queries"], segments=g[p + "segments"])
    feat = sk.compute_features(wl, sk.ControllerConfig())
    np.testing.assert_allclose(feat.u_hat, g[p + "u_hat"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(feat.s_hat, g[p + "s_hat"], rtol=1e-9, atol=1e-12)
    assert abs(feat.r_q - float(g[p + "r_q"])) <= 1e-12 * abs(float(g[p + "r_q"]))


def test_recon_negative_control_matches_angle_with_tax(sk):
    """decode.py:195-217 (reference test_decode.py:100-113): the reconstruct-
    then-dot path gives the angle path's numbers while the meter carries the
    exact densification tax n * d * 2 bytes each way on top."""
    rng = np.random.default_rng(5)
    L, H, T, d, P = 1, 2, 300, 64, 128
    tl = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)]
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    keys = rng.standard_normal((L, H, T, d))
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    r, ang = O.encode_batch(keys.reshape(-1, d))
    r, ang = r.reshape(L, H, T), ang.reshape(L, H, T, d - 1)
    tier = rng.choice([0, 1, 2, 3], (L, H, T)).astype(np.int16)
    z = (tier != 0).astype(np.int8)
    prot = np.zeros((L, H, T), bool)

    def build():
        return sk.pack_pages_arrays(sk.TierAssignment(z, tier, prot), r, ang, vals, tiers, P)

    st_a, st_r = build(), build()
    q = rng.standard_normal(d) * 3
    st_a.meter.reset()
    st_r.meter.reset()
    la = sk.angle_logits(q, st_a, 0, 1)
    lr = sk.recon_logits(q, st_r, 0, 1)
    n = int(z[0, 1].sum())
    assert la.shape == lr.shape == (n,)
    assert np.max(np.abs(la - lr) / np.maximum(1, np.abs(lr))) < 1e-4
    ost = O.pack_pages(tl, z, tier, prot, r, ang, vals, P)
    rq, qf = O.query_features(q[None])
    want, want_out = O.head_attend(ost, 0, 1, rq[0], qf[0])
    assert np.max(np.abs(lr - want) / np.maximum(1, np.abs(want))) < LOGIT_TOL
    snap = st_r.meter.snapshot()
    assert snap["dense_k_write"] == snap["dense_k_read"] == n * d * 2
    assert st_r.meter.total_bytes == st_a.meter.total_bytes + n * d * 2 * 2
    lg, out, cnt, _ = sk.decode._head_attend("recon", st_r, 0, 1, q)
    assert cnt == n and np.max(np.abs(out - want_out)) / np.max(np.abs(want_out)) < OUT_TOL


def test_decode_margins_for_the_gate(sk):
    """Per (group, q-head) top-1 minus top-2 logit from the decode kernel (the
    gate input, gate.py:50-56 on decode.py:433-436 logits) vs the oracle's
    logits; empty and one-item heads give +inf; outputs are unchanged."""
    import torch
    from paper_2605_18856_b200 import gate

    wl = sk.synth.generate(1, 1, 3, 4, 2000, 64, seed=7)
    tiers = table(sk, [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)])
    st = sk.PagedStore(tiers, 1, 3, 64, 64, 128, capacity_tokens=2000)
    n = wl.groups * wl.tokens
    rng = np.random.default_rng(4)
    tier = rng.choice([0, 1, 2, 3], n, p=[0.1, 0.4, 0.4, 0.1]).astype(np.int16)
    tier[wl.tokens: 2 * wl.tokens] = 0      # group 1: empty
    tier[2 * wl.tokens: 3 * wl.tokens] = 0  # group 2: a single item
    tier[2 * wl.tokens + 17] = 2
    radii = torch.empty(n, dtype=torch.float64, device="cuda")
    from paper_2605_18856_b200 import _lib
    _lib.check(_lib.lib().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, 64,
                                             radii.data_ptr(), _lib.stream_ptr()))
    sk.pack_device(st, keys=wl.keys.view(-1, 64), radii=radii, values=wl.values.view(-1, 64),
                   z=(tier != 0).astype(np.int8), tier=tier, protect=np.zeros(n, np.uint8),
                   tokens=wl.tokens)
    for grid in (1, 5, 148):
        plan = sk.plan_store(st, grid=grid, units_per_cta=1)
        margins = torch.full((3 * 4,), -1.0, dtype=torch.float32, device="cuda")
        out = sk.ada_decode(st, wl.queries, plan, margins=margins)
        ref = sk.ada_decode(st, wl.queries, plan)
        assert torch.allclose(out, ref, rtol=1e-6, atol=1e-6)
        m = margins.view(3, 4).cpu().numpy()
        lg, _ = sk.decode.attend_heads(st, 0, 0, wl.queries[0].double().cpu().numpy())
        for g in range(4):
            want = gate.margin(lg[g])
            assert abs(m[0, g] - want) <= 2e-3 * max(1.0, np.abs(lg[g]).max()), (g, m[0, g], want)
        assert np.all(np.isinf(m[1])) and np.all(np.isinf(m[2]))


@pytest.mark.parametrize("d,P,G", [(128, 256, 1), (128, 256, 5), (128, 256, 8), (64, 128, 8),
                                   (64, 128, 3)])
def test_specialised_tiles_all_gqa_widths(sk, d, P, G):
    """The specialised tile kernels (d in {64, 128}, P % 128 == 0) for every
    GQA width class (GP = 1..4: G = 1, 3, 5, 8 -- Llama 4, Qwen 5, gpt-oss 8)
    and every panel tier, against the oracle on identical inputs."""
    rng = np.random.default_rng(d * 100 + G)
    tl = [tuple(t) for t in sk.synth.PANEL_TIERS]
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    L, H, T = 1, 2, 2 * P + 77
    keys = rng.standard_normal((L, H, T, d)) * rng.uniform(0.5, 2.0, (L, H, T, 1))
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    r, ang = O.encode_batch(keys.reshape(-1, d))
    r, ang = r.reshape(L, H, T), ang.reshape(L, H, T, d - 1)
    tier = rng.choice([0, 1, 2, 3, 4, 5, 6], (L, H, T)).astype(np.int16)
    z = (tier != 0).astype(np.int8)
    prot = np.zeros((L, H, T), bool)
    st = sk.pack_pages_arrays(sk.TierAssignment(z, tier, prot), r, ang, vals, tiers, P)
    ost = O.pack_pages(tl, z, tier, prot, r, ang, vals, P)
    for h in range(H):
        q = rng.standard_normal((G, d)) * 3
        lg, out = sk.decode.attend_heads(st, 0, h, q)
        rq, qf = O.query_features(q)
        for g in range(G):
            want_lg, want_out = O.head_attend(ost, 0, h, rq[g], qf[g])
            assert_attend_close(lg[g], out[g], want_lg, want_out)


def test_errors_follow_the_reference(sk):
    """The drop-in raises what the reference raises for the same misuse:
    KeyError for unknown heads / missing states (store.py:286-287, :442-445),
    ValueError for a retained state on the drop tier (store.py:450-451) and
    for a query of the wrong width."""
    tiers = table(sk, [(0, 0, 0, 0), (1, 4, 6, 0)])
    L, H, T, d = 1, 2, 64, 8
    rng = np.random.default_rng(3)
    r, a = O.encode_batch(rng.standard_normal((L * H * T, d)))
    r, a = r.reshape(L, H, T), a.reshape(L, H, T, d - 1)
    vals = rng.standard_normal((L, H, T, d))
    z = np.ones((L, H, T), np.int8)
    prot = np.zeros((L, H, T), bool)
    st = sk.pack_pages_arrays(sk.TierAssignment(z, z.astype(np.int16), prot), r, a, vals,
                              tiers, 32)
    with pytest.raises(KeyError):
        list(st.stream_pages(0, H))
    with pytest.raises(KeyError):
        sk.angle_logits(np.ones(d), st, 1, 0)
    with pytest.raises(ValueError):
        sk.angle_logits(np.ones(d + 1), st, 0, 0)
    with pytest.raises(KeyError):  # key arrays shorter than the assignment
        sk.pack_pages_arrays(sk.TierAssignment(z, z.astype(np.int16), prot), r[:, :, :T - 1],
                             a[:, :, :T - 1], vals, tiers, 32)
    with pytest.raises(ValueError):  # retained state on the drop tier
        sk.pack_pages_arrays(sk.TierAssignment(z, np.zeros((L, H, T), np.int16), prot), r, a,
                             vals, tiers, 32)


# ---------------------------------------------------------------------------
# decode steps with appends (decode.py:415-498)
# ---------------------------------------------------------------------------

def oracle_rollout(ost, qs, ks, vs, u_hat, s_hat, r_q, tl, eps, lam, gate_cfg, prefill, omega):
    """Reference decode loop restated on the oracle store: per step and
    (l, h) attention + margins, best tier of the new key, hysteretic gate,
    append.  GQA: danger = max over the query heads.  Returns per-step
    outputs, tiers, protect flags, modes."""
    L, H = ost.layers, ost.heads
    d = ost.d
    mode = np.ones((L, H), np.int8)
    logs = []
    for t in range(len(qs)):
        outs = np.zeros((L, H, qs.shape[3], ost.d_v))
        tiers = np.zeros((L, H), np.int16)
        prots = np.zeros((L, H), np.uint8)
        for l in range(L):
            for h in range(H):
                q = qs[t, l, h]
                rq, qf = O.query_features(q)
                margins = []
                for g in range(q.shape[0]):
                    lg, out = O.head_attend(ost, l, h, rq[g], qf[g])
                    outs[l, h, g] = out
                    margins.append(math.inf if lg.size < 2 else float(np.diff(np.sort(lg)[-2:])[0]))
                k = ks[t, l, h]
                r = float(O.pairwise_norm(k[None])[0])
                ang = O.angles_from_unit((k / (r + O.NORM_EPS))[None])[0]
                tid = O.score_one(r, u_hat[l, h], s_hat[l, h], r_q, omega, 1.0, 1.0, tl, eps, lam,
                                  d)[0]
                prot = False
                if gate_cfg is not None:
                    probe = tid if tid != 0 else tl[-1][0]
                    et, er_rel = eps[probe]
                    r_max = max((ost.pages[i].scale for i in ost.pointer[(l, h)]), default=0.0)
                    er = er_rel * r_max
                    danger = 0.0
                    for g in range(q.shape[0]):
                        qn = float(O.pairwise_norm(q[g][None])[0])
                        bound = gate_cfg.alpha * ((qn / math.sqrt(d)) * (r_max * et + er + er * et))
                        m = margins[g]
                        dg = 0.0 if math.isinf(m) else min(bound / (m + 1e-9), 10.0)
                        danger = max(danger, dg)
                    if danger >= gate_cfg.tau_prot:
                        mode[l, h] = 2
                    elif danger <= gate_cfg.tau_drop:
                        mode[l, h] = 0
                    if mode[l, h] == 2:
                        tid, prot = tl[-1][0], True
                tiers[l, h], prots[l, h] = tid, prot
                ost.append_item(l, h, r, ang, vs[t, l, h], tid, prot, token_id=prefill + t)
        logs.append((outs, tiers, prots, mode.copy()))
    return logs


@pytest.mark.parametrize("use_gate", [False, True])
def test_decode_steps_with_appends_match_oracle_rollout(sk, use_gate):
    """DecodeStepper (live decode + margins -> gate -> append, one CUDA graph
    per step) vs the oracle restatement of the reference decode loop:
    outputs within tolerance, per-step tier / protect / gate decisions and
    the final SPHKV1 store bytes identical."""
    import torch

    rng = np.random.default_rng(21 + use_gate)
    L, H, G, T, d, P, N = 2, 2, 4, 700, 64, 128, 12
    tl = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)]
    eps = {1: (0.08, 0.02), 2: (0.02, 0.005), 3: (0.001, 0.0003)}
    tiers = table(sk, tl, eps=[eps[1], eps[2], eps[3]])
    keys = rng.standard_normal((L, H, T, d))
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    r, ang = O.encode_batch(keys.reshape(-1, d))
    r, ang = r.reshape(L, H, T), ang.reshape(L, H, T, d - 1)
    tier = rng.choice([0, 1, 2, 3], (L, H, T), p=[0.2, 0.5, 0.2, 0.1]).astype(np.int16)
    z = (tier != 0).astype(np.int8)
    prot = np.zeros((L, H, T), bool)
    st = sk.pack_pages_arrays(sk.TierAssignment(z, tier, prot), r, ang, vals, tiers, P,
                              append_tokens=64)
    ost = O.pack_pages(tl, z, tier, prot, r, ang, vals, P)
    u_hat = rng.uniform(0.2, 1.0, (L, H))
    s_hat = rng.uniform(0.0, 0.8, (L, H))
    r_q, lam, omega = 30.0, 3e-4, 1.0
    qs = (rng.standard_normal((N, L, H, G, d)) * 3).astype(np.float32).astype(np.float64)
    ks = rng.standard_normal((N, L, H, d))
    ks[:, 0, 1] *= 3.0  # outlier-sized keys: page scale / new-page rule
    ks = ks.astype(np.float32).astype(np.float64)  # the device step takes fp32 keys
    vs = rng.standard_normal((N, L, H, d)).astype(np.float16).astype(np.float64)
    gate_cfg = sk.GateConfig(tau_drop=0.02, tau_prot=0.2) if use_gate else None
    want = oracle_rollout(ost, qs, ks, vs, u_hat, s_hat, r_q, tl, eps, lam, gate_cfg, T, omega)
    stp = sk.DecodeStepper(st, G, u_hat, s_hat, r_q, lam=lam, omega=omega, gate_cfg=gate_cfg)
    stp.capture()
    for t in range(N):
        out = stp.step(torch.as_tensor(qs[t].reshape(-1, G, d), dtype=torch.float32, device="cuda"),
                       torch.as_tensor(ks[t].reshape(-1, d), dtype=torch.float32, device="cuda"),
                       torch.as_tensor(vs[t].reshape(-1, d), dtype=torch.float16, device="cuda"),
                       T + t)
        w_out, w_tier, w_prot, w_mode = want[t]
        got = out.double().cpu().numpy().reshape(L, H, G, d)
        den = np.max(np.abs(w_out))
        assert np.max(np.abs(got - w_out)) / den < OUT_TOL
        assert np.array_equal(stp.tier.cpu().numpy().reshape(L, H), w_tier)
        assert np.array_equal(stp.prot.cpu().numpy().reshape(L, H), w_prot)
        if use_gate:
            assert np.array_equal(stp.mode.cpu().numpy().reshape(L, H), w_mode)
    stp.finish()
    assert st.to_bytes() == ost.to_bytes()
    st.check_invariants()
    if use_gate:  # the gate must have acted somewhere for the test to mean anything
        assert any(np.any(w[2]) for w in want) or any(np.any(w[3] == 0) for w in want)
