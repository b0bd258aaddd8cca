"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side schema (tiers, config) behaves like the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sphkv_b200.h")
LIB = os.path.join(ROOT, "paper_2605_18856_b200", "libsphkv_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(sphkv_\w+)\s*\(", text,
                                 flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ("sphkv_ada_decode", "sphkv_lse_merge", "sphkv_rdr_allocate_greedy",
              "sphkv_pack_pages", "sphkv_append", "sphkv_encode", "sphkv_rdr_score"):
        assert s in syms


def test_library_loads_and_exports_every_symbol():
    import __graft_entry__

    __graft_entry__.build()  # incremental: rebuilds only when sources changed
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    lib.sphkv_abi_version.restype = ctypes.c_int
    assert lib.sphkv_abi_version() == 1
    lib.sphkv_partial_floats.restype = ctypes.c_int64
    assert lib.sphkv_partial_floats(4, 128) == 4 * 130


def test_product_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_18856_b200 as sk

    with pytest.raises(RuntimeError):
        sk.to_spherical(np.ones(4))


def test_tier_schema_like_reference():
    import paper_2605_18856_b200 as sk

    assert sk.rate_bits(sk.TierSpec(1, 4, 8, 8), 64) == 268
    assert sk.rate_bits(sk.TierSpec(0, 0, 0, 0), 64) == 0
    with pytest.raises(ValueError):
        sk.TierSpec(0, 1, 0, 0)
    with pytest.raises(ValueError):
        sk.TierSpec(1, 0, 4, 0)
    t = sk.TierTable((sk.TierSpec(0, 0, 0, 0), sk.TierSpec(1, 4, 4, 0), sk.TierSpec(2, 4, 4, 0)))
    with pytest.raises(ValueError):
        t.validate_rates(8)
    text = "tier 0 0 0 0\ntier 1 2 4 8\ntier 2 4 6 8"
    assert sk.TierTable.parse(text).serialize() == text
    with pytest.raises(ValueError):
        sk.TierTable.parse("tier 1 2")


def test_config_roundtrip_and_fail_closed():
    from paper_2605_18856_b200 import config

    cfg = config.RunConfig()
    text = config.emit(cfg)
    assert config.parse(text) == cfg
    assert config.emit(config.parse(text)) == text
    panel = open(os.path.join(ROOT, "tests", "golden", "panel.cfg")).read()
    p = config.parse(panel)
    assert p.workload.page_size == 1024 and p.controller.lam == 3e-5
    assert [t.angle_bits for t in p.tiers.tiers] == [0, 2, 4, 6, 7, 12, 15]
    assert config.parse(config.emit(p)) == p
    for bad in ("[workload]\nwarp_factor = 9\n", "[mystery]\nx = 1\n", "stray = 1\n"):
        with pytest.raises(ValueError):
            config.parse(bad)


def test_resident_closed_form_matches_oracle():
    """synth.resident_total (used for budget bisection) == the oracle store accounting."""
    from oracle import sphkv_oracle as O
    from paper_2605_18856_b200 import synth
    import paper_2605_18856_b200 as sk

    rng = np.random.default_rng(0)
    tl = [tuple(x) for x in synth.PANEL_TIERS]
    L, H, T, d, P = 1, 3, 1000, 16, 64
    tier = rng.integers(0, 7, (L, H, T)).astype(np.int16)
    z = (tier != 0).astype(np.int8)
    radii = rng.uniform(0.5, 2, (L, H, T))
    ang = rng.uniform(0, 1, (L, H, T, d - 1))
    st = O.pack_pages(tl, z, tier, np.zeros((L, H, T), bool), radii, ang,
                      np.zeros((L, H, T, d)), P)
    counts = np.stack([[np.sum(tier[0, h] == t[0]) for t in tl] for h in range(H)])
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in tl))
    assert synth.resident_total(counts, tiers, d, d, P, H) == st.resident_breakdown()["total"]
