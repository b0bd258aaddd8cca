"""Spherical key codec, B200 edition (drop-in for sphkv.codec, pkg/src/sphkv/codec.py).

Host side: the tier schema (TierSpec / TierTable, rate model, text form,
calibration) -- configuration, not compute.  Device side: the encoder and
quantizers run as sm_100a kernels through libsphkv_b200 (`sphkv_encode`,
`sphkv_quantize_angles`); numpy arrays in, numpy arrays out, like the
reference.  Bit-exactness contract: codes and radii equal
the reference's on identical fp64 inputs (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

DROP_TIER_ID = 0
MAX_CODE_BITS = 53          # codec.py:37-39 (schema limit)
DEVICE_MAX_CODE_BITS = 16   # kernel contract
TWO_PI = 2.0 * math.pi
_NORM_EPS = 1e-12


@dataclass(frozen=True)
class SphericalKey:
    """Radius plus (d-1) hyperspherical angles (codec.py:56-70)."""

    radius: float
    angles: np.ndarray

    def __post_init__(self):
        if self.radius < 0:
            raise ValueError(f"radius must be nonnegative, got {self.radius}")
        object.__setattr__(self, "angles", np.asarray(self.angles, dtype=np.float64))

    @property
    def dim(self) -> int:
        return self.angles.shape[0] + 1


@dataclass(frozen=True)
class TierSpec:
    """Bit widths of one tier; id 0 is the zero-rate drop tier (codec.py:73-98)."""

    id: int
    angle_bits: int
    radius_bits: int
    meta_bits: int

    def __post_init__(self):
        widths = (self.angle_bits, self.radius_bits, self.meta_bits)
        if self.id == DROP_TIER_ID and any(widths):
            raise ValueError("drop tier must have zero bit widths")
        if self.id != DROP_TIER_ID and (self.angle_bits < 1 or self.radius_bits < 1):
            raise ValueError(f"tier {self.id}: angle_bits and radius_bits must be >= 1")
        for name, b in zip(("angle_bits", "radius_bits", "meta_bits"), widths):
            if not 0 <= b <= MAX_CODE_BITS:
                raise ValueError(f"tier {self.id}: {name}={b} outside [0, {MAX_CODE_BITS}]")

    @property
    def is_drop(self) -> bool:
        return self.id == DROP_TIER_ID


def rate_bits(tier: TierSpec, d: int) -> int:
    """R(t) = (d-1) b_angle + b_radius + b_meta; 0 for drop (codec.py:101-107)."""
    if d < 2:
        raise ValueError(f"head dimension must be >= 2, got {d}")
    return 0 if tier.is_drop else (d - 1) * tier.angle_bits + tier.radius_bits + tier.meta_bits


@dataclass
class TierTable:
    """Ordered tier set, drop first, with calibrated eps constants (codec.py:110-196)."""

    tiers: tuple
    eps_theta: dict = field(default_factory=dict)
    eps_r: dict = field(default_factory=dict)

    def __post_init__(self):
        self.tiers = tuple(self.tiers)
        if not self.tiers or not self.tiers[0].is_drop:
            raise ValueError("tier table must start with the drop tier (id 0)")
        ids = [t.id for t in self.tiers]
        if ids != sorted(ids) or len(set(ids)) != len(ids):
            raise ValueError(f"tier ids must be unique and ascending, got {ids}")

    def __iter__(self):
        return iter(self.tiers)

    @property
    def non_drop(self):
        return self.tiers[1:]

    @property
    def max_tier(self) -> TierSpec:
        if len(self.tiers) < 2:
            raise ValueError("tier table has no non-drop tiers")
        return self.tiers[-1]

    def spec_for(self, tier_id: int) -> TierSpec:
        for t in self.tiers:
            if t.id == tier_id:
                return t
        raise KeyError(f"unknown tier id {tier_id}")

    def rate_bits(self, tier_id: int, d: int) -> int:
        return rate_bits(self.spec_for(tier_id), d)

    def validate_rates(self, d: int) -> None:
        rates = [rate_bits(t, d) for t in self.non_drop]
        if any(b <= a for a, b in zip(rates, rates[1:])):
            raise ValueError(f"tier rates not strictly increasing at d={d}: {rates}")

    @property
    def calibrated(self) -> bool:
        return all(t.id in self.eps_theta for t in self.non_drop)

    def distortion_constants(self, tier_id: int):
        if tier_id == DROP_TIER_ID:
            return 1.0, 1.0
        if tier_id not in self.eps_theta:
            raise KeyError(f"tier {tier_id} is not calibrated")
        return self.eps_theta[tier_id], self.eps_r[tier_id]

    def calibrate(self, sample, seed: int, queries_per_key: int = 1) -> None:
        for t in self.non_drop:
            self.eps_theta[t.id], self.eps_r[t.id] = calibrate_distortion(
                t, sample, seed, queries_per_key)

    def serialize(self) -> str:
        return "\n".join(f"tier {t.id} {t.angle_bits} {t.radius_bits} {t.meta_bits}"
                         for t in self.tiers)

    @classmethod
    def parse(cls, text: str) -> "TierTable":
        specs = []
        for raw in text.strip().splitlines():
            line = raw.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split()
            if len(parts) != 5 or parts[0] != "tier":
                raise ValueError(f"bad tier line: {line!r}")
            specs.append(TierSpec(*(int(p) for p in parts[1:])))
        return cls(tuple(specs))


@dataclass(frozen=True)
class AngleCode:
    codes: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "codes", np.asarray(self.codes, dtype=np.uint64))


@dataclass(frozen=True)
class RadiusCode:
    code: int


# ---------------------------------------------------------------------------
# device encoder / quantizer
# ---------------------------------------------------------------------------

def _dev(arr, dtype):
    import torch

    return torch.as_tensor(np.ascontiguousarray(arr, dtype=dtype), device="cuda")


def encode_batch(keys: np.ndarray):
    """Batched to_spherical on the GPU: (n, d) -> radii (n,), angles (n, d-1).

    Radii use numpy's pairwise summation order (np.linalg.norm(k, axis=1))."""
    import torch

    l = _lib.require_gpu()
    keys = np.asarray(keys, dtype=np.float64)
    if keys.ndim != 2:
        raise ValueError("keys must be (n, d)")
    n, d = keys.shape
    if d < 2:
        raise ValueError(f"need d >= 2, got {d}")
    k = _dev(keys, np.float64)
    r = torch.empty(n, dtype=torch.float64, device="cuda")
    a = torch.empty((n, d - 1), dtype=torch.float64, device="cuda")
    _lib.check(l.sphkv_encode(k.data_ptr(), _lib.F64, n, d, r.data_ptr(), a.data_ptr(),
                              _lib.stream_ptr()))
    return r.cpu().numpy(), a.cpu().numpy()


def to_spherical(k: np.ndarray) -> SphericalKey:
    """Dense vector -> SphericalKey (codec.py:222-236), on the device."""
    k = np.asarray(k, dtype=np.float64)
    if k.ndim != 1:
        raise ValueError("to_spherical takes one vector")
    if k.shape[0] < 2:
        raise ValueError(f"need d >= 2, got {k.shape[0]}")
    r, a = encode_batch(k[None, :])
    return SphericalKey(float(r[0]), a[0])


def angles_from_unit(u: np.ndarray) -> np.ndarray:
    """Angles of unit rows (codec.py:239-257): the encoder on r = 1 inputs."""
    import torch

    l = _lib.require_gpu()
    u = np.asarray(u, dtype=np.float64)
    n, d = u.shape
    ud = _dev(u, np.float64)
    a = torch.empty((n, d - 1), dtype=torch.float64, device="cuda")
    _lib.check(l.sphkv_angles_from_unit(ud.data_ptr(), n, d, a.data_ptr(), _lib.stream_ptr()))
    return a.cpu().numpy()


def quantize_angles(angles: np.ndarray, bits: int) -> np.ndarray:
    """quantize_angles (codec.py:326-340) on the device; uint64 codes."""
    import torch

    if bits < 1 or bits > 31:
        raise ValueError(f"device quantizer supports 1..31 bits, got {bits}")
    l = _lib.require_gpu()
    angles = np.asarray(angles, dtype=np.float64)
    shape = angles.shape
    flat = angles.reshape(-1, shape[-1])
    a = _dev(flat, np.float64)
    out = torch.empty(flat.shape, dtype=torch.int32, device="cuda")
    _lib.check(l.sphkv_quantize_angles(a.data_ptr(), flat.shape[0], flat.shape[1], bits,
                                       out.data_ptr(), _lib.stream_ptr()))
    return out.cpu().numpy().view(np.uint32).astype(np.uint64).reshape(shape)


def _polar_step(bits: int) -> float:
    return math.pi / float((1 << bits) - 1) if bits >= 1 else math.pi


def _circular_step(bits: int) -> float:
    return TWO_PI / float(1 << bits)


def dequantize_angles(codes: np.ndarray, bits: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint64)
    out = np.empty(codes.shape, dtype=np.float64)
    dm1 = codes.shape[-1]
    if dm1 > 1:
        out[..., : dm1 - 1] = codes[..., : dm1 - 1].astype(np.float64) * _polar_step(bits)
    out[..., dm1 - 1] = codes[..., dm1 - 1].astype(np.float64) * _circular_step(bits)
    return out


def quantize_radius(r: float, scale: float, bits: int) -> int:
    levels = (1 << bits) - 1
    return int(round(min(max(r / scale, 0.0), 1.0) * levels))


def dequantize_radius(code: int, scale: float, bits: int) -> float:
    levels = (1 << bits) - 1
    if not 0 <= code <= levels:
        raise ValueError(f"radius code {code} out of range for {bits} bits")
    return code / levels * scale


def encode_key(s: SphericalKey, t: TierSpec, radius_scale: float):
    """Quantize one key at tier t against a page radius scale (codec.py:365-377)."""
    if t.is_drop:
        raise ValueError("cannot encode at the drop tier")
    if radius_scale <= 0:
        raise ValueError("radius_scale must be positive")
    if s.radius > radius_scale * (1 + 1e-12):
        raise ValueError(f"radius {s.radius} exceeds page scale {radius_scale} (page-packing bug)")
    a = quantize_angles(s.angles[None, :], t.angle_bits)[0]
    return AngleCode(a), RadiusCode(quantize_radius(s.radius, radius_scale, t.radius_bits))


def decode_key(a: AngleCode, r: RadiusCode, t: TierSpec, radius_scale: float) -> SphericalKey:
    if t.is_drop:
        raise ValueError("cannot decode the drop tier")
    if a.codes.max(initial=0) >= (1 << t.angle_bits):
        raise ValueError("angle code out of range (corrupt stream)")
    return SphericalKey(dequantize_radius(r.code, radius_scale, t.radius_bits),
                        dequantize_angles(a.codes, t.angle_bits))


def angular_features(angles: np.ndarray) -> np.ndarray:
    """Feature rows of the recurrence (codec.py:459-477) -- host helper for
    query-side inspection; the device computes them inside the decode kernel."""
    angles = np.atleast_2d(np.asarray(angles, dtype=np.float64))
    n, dm1 = angles.shape
    c, s = np.cos(angles), np.sin(angles)
    prods = np.cumprod(s, axis=1)
    out = np.empty((n, dm1 + 1))
    out[:, 0] = c[:, 0]
    out[:, 1:dm1] = prods[:, : dm1 - 1] * c[:, 1:]
    out[:, dm1] = prods[:, dm1 - 1]
    return out


def cos_from_angles(q_angles, k_angles) -> float:
    fq = angular_features(np.asarray(q_angles)[None])[0]
    fk = angular_features(np.asarray(k_angles)[None])[0]
    return float(fq @ fk)


def cos_from_codes(q_angles, k_code: AngleCode, t: TierSpec) -> float:
    if t.is_drop:
        raise ValueError("drop tier carries no angle code")
    return cos_from_angles(q_angles, dequantize_angles(k_code.codes, t.angle_bits))


def from_spherical(s: SphericalKey) -> np.ndarray:
    """Densification primitive (codec.py:260-267); never used by the decode path."""
    return s.radius * angular_features(s.angles[None])[0]


# ---------------------------------------------------------------------------
# calibration (host setup step, codec.py:485-534)
# ---------------------------------------------------------------------------

def calibrate_distortion(t: TierSpec, sample, seed: int, queries_per_key: int = 1):
    """RMS distortion constants of tier t on a key sample (setup, not hot path).

    Query angles come from the device encoder; the recurrence differences
    are evaluated in fp64 on the host as in the reference."""
    if not sample:
        raise ValueError("calibration sample must be nonempty")
    if t.is_drop:
        raise ValueError("drop tier is not calibrated")
    rng = np.random.default_rng(seed)
    d = sample[0].dim
    k_angles = np.stack([s.angles for s in sample])
    k_dec = dequantize_angles(quantize_angles(k_angles, t.angle_bits), t.angle_bits)
    sq_acc, n_terms = 0.0, 0
    for _ in range(queries_per_key):
        q = rng.standard_normal((len(sample), d))
        q /= np.linalg.norm(q, axis=1, keepdims=True) + _NORM_EPS
        qa = angles_from_unit(q)
        exact = np.sum(angular_features(qa) * angular_features(k_angles), axis=1)
        coded = np.sum(angular_features(qa) * angular_features(k_dec), axis=1)
        sq_acc += float(np.sum((exact - coded) ** 2))
        n_terms += len(sample)
    eps_theta = math.sqrt(sq_acc / n_terms)
    radii = np.array([s.radius for s in sample])
    scale = float(radii.max()) + _NORM_EPS
    codes = np.array([quantize_radius(r, scale, t.radius_bits) for r in radii])
    decoded = codes / float((1 << t.radius_bits) - 1) * scale
    eps_r = math.sqrt(float(np.mean(((decoded - radii) / scale) ** 2)))
    return eps_theta, eps_r
