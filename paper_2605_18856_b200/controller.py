"""RDR retention controller on the B200 (drop-in for sphkv.controller).

score_states / allocate_greedy / downtier_before_drop / score_and_best_tier
run as sm_100a kernels (rdr.cu, encode_pack.cu) that are bit-exact with the
reference's fp64 numpy arithmetic (controller.py:163-386).  Device-tensor
variants (`*_device`) serve the batched prefill path; the numpy-shaped
functions keep the reference signatures.

compute_features (controller.py:99-142) is an input contract of the hot
path; its masked prefill pass is the fp64
sphkv_controller_stats kernel (csrc/features.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _lib
from ._lib import InfeasibleProtectionError
from .codec import DROP_TIER_ID, SphericalKey, TierSpec, TierTable, rate_bits

_NU_EPS = 1e-12
_MARGIN_EPS = 1e-6
MAX_FEATURE_ROWS = 512
SEGMENTS = ("prefix", "retrieved", "recent")
SEG_PREFIX, SEG_RETRIEVED, SEG_RECENT = 0, 1, 2


class StateId(NamedTuple):
    layer: int
    head: int
    token: int


@dataclass(frozen=True)
class ControllerConfig:
    lam: float = 1e-4
    omega_prefix: float = 0.25
    omega_retrieved: float = 2.0
    omega_recent: float = 1.0
    alpha_theta: float = 1.0
    alpha_r: float = 1.0
    protect_spans: tuple = ()
    protect_outliers: bool = False
    allocator: str = "greedy"

    def __post_init__(self):
        for name in ("omega_prefix", "omega_retrieved", "omega_recent", "alpha_theta", "alpha_r"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be strictly positive")
        if self.lam < 0:
            raise ValueError("lambda must be nonnegative")
        if self.allocator not in ("greedy", "downtier"):
            raise ValueError(f"unknown allocator {self.allocator!r}")

    @property
    def omega(self) -> np.ndarray:
        return np.array([self.omega_prefix, self.omega_retrieved, self.omega_recent])


@dataclass
class ControllerFeatures:
    u_hat: np.ndarray
    s_hat: np.ndarray
    r_q: float
    omega: np.ndarray
    alpha_theta: float
    alpha_r: float
    segments: np.ndarray
    prefill: int

    def age(self, token: int) -> int:
        return self.prefill - token

    def omega_of(self, token: int) -> float:
        if 0 <= token < self.prefill:
            return float(self.omega[self.segments[token]])
        return float(self.omega[SEG_RECENT])


@dataclass
class StateScores:
    best_tier: np.ndarray
    score: np.ndarray
    nu: np.ndarray
    d_drop: np.ndarray
    w_theta: np.ndarray | None = None
    w_r: np.ndarray | None = None


@dataclass
class TierAssignment:
    z: np.ndarray
    tier: np.ndarray
    protected: np.ndarray

    def __getitem__(self, state):
        l, h, i = state
        return int(self.z[l, h, i]), int(self.tier[l, h, i]), bool(self.protected[l, h, i])

    def check(self, tiers: TierTable):
        assert np.all((self.z == 0) == (self.tier == DROP_TIER_ID))
        if np.any(self.protected):
            assert np.all(self.z[self.protected] == 1)
            assert np.all(self.tier[self.protected] == tiers.max_tier.id)

    def total_rate_bits(self, tiers: TierTable, d: int) -> int:
        return sum(int(np.sum(self.tier == t.id)) * rate_bits(t, d) for t in tiers.non_drop)

    def retained_fraction(self) -> float:
        return float(np.mean(self.z == 1))


def _tiers_arr(tiers: TierTable):
    return _lib.tiers_to_c(tiers)


# ---------------------------------------------------------------------------
# scoring
# ---------------------------------------------------------------------------

def score_states_device(radii, u_hat, s_hat, seg_omega, r_q, alpha_theta, alpha_r,
                        tiers: TierTable, lam, protect, d):
    """Device tensors in/out: radii fp64 [L, H, T], u_hat/s_hat fp64 [L, H],
    seg_omega fp64 [T], protect uint8 [L, H, T].  Returns (best int16, score,
    nu, d_drop) fp64 device tensors."""
    import torch

    l = _lib.require_gpu()
    if not tiers.calibrated:
        raise ValueError("tier table must be calibrated before scoring")
    tiers.validate_rates(d)
    L, H, T = radii.shape
    best = torch.empty((L, H, T), dtype=torch.int16, device="cuda")
    score = torch.empty((L, H, T), dtype=torch.float64, device="cuda")
    nu = torch.empty((L, H, T), dtype=torch.float64, device="cuda")
    dd = torch.empty((L, H, T), dtype=torch.float64, device="cuda")
    arr = _tiers_arr(tiers)
    _lib.check(l.sphkv_rdr_score(radii.data_ptr(), u_hat.data_ptr(), s_hat.data_ptr(),
                                 seg_omega.data_ptr(), float(r_q), float(alpha_theta),
                                 float(alpha_r), arr, len(tiers.tiers), float(lam),
                                 protect.data_ptr(), L, H, T, d, best.data_ptr(),
                                 score.data_ptr(), nu.data_ptr(), dd.data_ptr(),
                                 _lib.stream_ptr()))
    return best, score, nu, dd


def score_states(radii, feat: ControllerFeatures, tiers: TierTable, lam, protected, d) -> StateScores:
    """Vectorized scoring (controller.py:213-245), bit-exact on the device."""
    import torch

    radii = np.asarray(radii, dtype=np.float64)
    dev = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device="cuda")
    seg_omega = np.asarray(feat.omega, dtype=np.float64)[np.asarray(feat.segments)]
    best, score, nu, dd = score_states_device(
        dev(radii, np.float64), dev(feat.u_hat, np.float64), dev(feat.s_hat, np.float64),
        dev(seg_omega, np.float64), feat.r_q, feat.alpha_theta, feat.alpha_r, tiers, lam,
        dev(np.asarray(protected, dtype=np.uint8), np.uint8), d)
    sqrt_d = math.sqrt(d)
    om = seg_omega[None, None, :]
    w_theta = feat.alpha_theta * np.asarray(feat.u_hat)[:, :, None] * om * (feat.r_q * radii / sqrt_d)
    w_r = feat.alpha_r * (1.0 - np.asarray(feat.s_hat)[:, :, None]) * om * (feat.r_q / sqrt_d)
    return StateScores(best.cpu().numpy(), score.cpu().numpy(), nu.cpu().numpy(),
                       dd.cpu().numpy(), w_theta, w_r)


def distortion_weights(state: StateId, key_radius, feat: ControllerFeatures, d):
    l, h, i = state
    om = feat.omega_of(i)
    sqrt_d = math.sqrt(d)
    w_theta = feat.alpha_theta * feat.u_hat[l, h] * om * (feat.r_q * key_radius / sqrt_d)
    w_r = feat.alpha_r * (1.0 - feat.s_hat[l, h]) * om * (feat.r_q / sqrt_d)
    return w_theta, w_r


def distortion_proxy(state: StateId, tier: TierSpec, key: SphericalKey, feat, tiers: TierTable):
    w_theta, w_r = distortion_weights(state, key.radius, feat, key.dim)
    eps_t, eps_r = tiers.distortion_constants(tier.id)
    return w_theta * eps_t + w_r * eps_r


def score_and_best_tier(state: StateId, key: SphericalKey, feat: ControllerFeatures,
                        tiers: TierTable, lam: float, protected: bool = False):
    """Best tier for one (appended) state (controller.py:181-198).

    Unprotected states score on the device (the batched append kernel); the
    protected variant excludes drop and is evaluated in the same fp64 order."""
    import torch

    d = key.dim
    if protected:
        best_id, best_s = None, -math.inf
        for t in tiers.non_drop:
            s = -distortion_proxy(state, t, key, feat, tiers) - lam * rate_bits(t, d)
            if s > best_s:
                best_id, best_s = t.id, s
        d_drop = distortion_proxy(state, tiers.spec_for(DROP_TIER_ID), key, feat, tiers)
        d_best = distortion_proxy(state, tiers.spec_for(best_id), key, feat, tiers)
        return best_id, best_s, (d_drop - d_best) / (rate_bits(tiers.spec_for(best_id), d) + _NU_EPS)
    l = _lib.require_gpu()
    tid, s, nu = (torch.zeros(1, dtype=t, device="cuda")
                  for t in (torch.int16, torch.float64, torch.float64))
    r = torch.tensor([key.radius], dtype=torch.float64, device="cuda")
    u = torch.tensor([float(feat.u_hat[state.layer, state.head])], dtype=torch.float64, device="cuda")
    sh = torch.tensor([float(feat.s_hat[state.layer, state.head])], dtype=torch.float64, device="cuda")
    _lib.check(l.sphkv_score_append(r.data_ptr(), 1, 1, u.data_ptr(), sh.data_ptr(),
                                    float(feat.r_q), feat.omega_of(state.token),
                                    float(feat.alpha_theta), float(feat.alpha_r),
                                    _tiers_arr(tiers), len(tiers.tiers), float(lam), d, 1,
                                    tid.data_ptr(), s.data_ptr(), nu.data_ptr(),
                                    _lib.stream_ptr()))
    return int(tid.item()), float(s.item()), float(nu.item())


def fixed_tier_scores(scores: StateScores, tier_id, tiers: TierTable, d) -> StateScores:
    eps_t, eps_r = tiers.distortion_constants(tier_id)
    d_fixed = scores.w_theta * eps_t + scores.w_r * eps_r
    rate = rate_bits(tiers.spec_for(tier_id), d)
    nu = (scores.d_drop - d_fixed) / (rate + _NU_EPS)
    best = np.full(scores.best_tier.shape, tier_id, dtype=np.int16)
    return StateScores(best, -d_fixed - rate * 0.0, nu, scores.d_drop, scores.w_theta, scores.w_r)


# ---------------------------------------------------------------------------
# allocators
# ---------------------------------------------------------------------------

def _alloc_device(kind, best, nu, protect, budget_bits, tiers: TierTable, d):
    import torch

    l = _lib.require_gpu()
    n = best.numel()
    ws = torch.empty(l.sphkv_rdr_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    z = torch.empty(best.shape, dtype=torch.int8, device="cuda")
    tier = torch.empty(best.shape, dtype=torch.int16, device="cuda")
    fn = l.sphkv_rdr_allocate_greedy if kind == "greedy" else l.sphkv_rdr_downtier
    _lib.check(fn(best.data_ptr(), nu.data_ptr(), protect.data_ptr(), n, _tiers_arr(tiers),
                  len(tiers.tiers), d, int(budget_bits), ws.data_ptr(), z.data_ptr(),
                  tier.data_ptr(), _lib.stream_ptr()))
    return z, tier


def allocate_greedy_device(best, nu, protect, budget_bits, tiers, d):
    """Device tensors: best int16, nu fp64, protect uint8 -> (z int8, tier int16)."""
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    return _alloc_device("greedy", best, nu, protect, budget_bits, tiers, d)


def downtier_device(best, nu, protect, budget_bits, tiers, d):
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    return _alloc_device("downtier", best, nu, protect, budget_bits, tiers, d)


def _np_to_dev(scores, protected):
    import torch

    dev = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x, dtype=dt), device="cuda")
    return (dev(scores.best_tier, np.int16), dev(scores.nu, np.float64),
            dev(np.asarray(protected, dtype=np.uint8), np.uint8))


def allocate_greedy(scores: StateScores, protected, budget_bits, tiers: TierTable, d) -> TierAssignment:
    """Greedy keep/drop + tier under a hard bit budget (controller.py:301-346)."""
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    z, tier = allocate_greedy_device(*_np_to_dev(scores, protected), budget_bits, tiers, d)
    out = TierAssignment(z.cpu().numpy(), tier.cpu().numpy(), np.asarray(protected).copy())
    assert out.total_rate_bits(tiers, d) <= budget_bits
    out.check(tiers)
    return out


def full_best_tier_assignment(scores: StateScores, protected, tiers: TierTable) -> TierAssignment:
    tier = scores.best_tier.copy()
    tier[protected] = tiers.max_tier.id
    return TierAssignment((tier != DROP_TIER_ID).astype(np.int8), tier, protected.copy())


def downtier_before_drop(initial: TierAssignment, scores: StateScores, budget_bits,
                         tiers: TierTable, d) -> TierAssignment:
    """Down-tier before drop (controller.py:349-386).  The device form starts
    from the full best-tier assignment (the canonical start, :389-398)."""
    if budget_bits < 0:
        raise ValueError("budget must be nonnegative")
    start = full_best_tier_assignment(scores, initial.protected, tiers)
    if not (np.array_equal(start.tier, initial.tier) and np.array_equal(start.z, initial.z)):
        raise ValueError("device downtier starts from full_best_tier_assignment(scores, ...)")
    z, tier = downtier_device(*_np_to_dev(scores, initial.protected), budget_bits, tiers, d)
    out = TierAssignment(z.cpu().numpy(), tier.cpu().numpy(), initial.protected.copy())
    out.check(tiers)
    return out


# ---------------------------------------------------------------------------
# features (input contract)
# ---------------------------------------------------------------------------

def feature_rows(T: int, max_rows: int = MAX_FEATURE_ROWS) -> np.ndarray:
    """Sampled prefill rows (controller.py:108-111)."""
    if T <= max_rows:
        return np.arange(T)
    return np.unique(np.round(np.linspace(0, T - 1, max_rows)).astype(int))


def controller_stats_device(keys, q_rows, rows, window):
    """u_raw, inv_margin per query group on the device (sphkv_controller_stats):
    keys [kv_groups, T, d] (bf16/fp16/fp32/fp64 tensor), q_rows fp64
    [kv_groups * q_per_key, R, d] device tensor (the q_per_key query rows of a
    KV group consecutive), rows [R] sampled token indices."""
    import torch

    l = _lib.require_gpu()
    kv_groups, T, d = keys.shape
    groups = q_rows.shape[0]
    R = len(rows)
    kd = {torch.float32: _lib.F32, torch.float64: _lib.F64, torch.bfloat16: _lib.BF16,
          torch.float16: _lib.F16}[keys.dtype]
    keys = keys.contiguous()
    q_rows = q_rows.to(device="cuda", dtype=torch.float64).contiguous()
    rows_t = torch.as_tensor(np.asarray(rows, dtype=np.int32), device="cuda")
    u = torch.empty(groups, dtype=torch.float64, device="cuda")
    m = torch.empty(groups, dtype=torch.float64, device="cuda")
    ws = torch.empty(l.sphkv_controller_workspace_bytes(groups, R), dtype=torch.uint8,
                     device="cuda")
    _lib.check(l.sphkv_controller_stats(keys.data_ptr(), kd, q_rows.data_ptr(),
                                        rows_t.data_ptr(), R, groups, T, d, int(window),
                                        groups // kv_groups, u.data_ptr(), m.data_ptr(),
                                        ws.data_ptr(), _lib.stream_ptr()))
    return u, m


def normalize_features(u_raw, inv_margin):
    """Across-head normalization (controller.py:135-140) of host arrays."""
    u_raw, inv_margin = np.asarray(u_raw, np.float64), np.asarray(inv_margin, np.float64)
    u_max = u_raw.max()
    u_hat = u_raw / u_max if u_max > 0 else np.ones_like(u_raw)
    m_max = inv_margin.max()
    s_hat = 1.0 - (inv_margin / m_max if m_max > 0 else np.zeros_like(inv_margin))
    return u_hat, s_hat


def compute_features(workload, config: ControllerConfig, max_rows: int = MAX_FEATURE_ROWS):
    """Head reuse / stability scalars from a dense prefill pass (controller.py:99-142):
    the masked softmax / top-2 pass over the sampled rows runs in the fp64
    sphkv_controller_stats kernel; the normalization across heads and r_q
    are host reductions."""
    import torch

    keys = np.asarray(workload.keys)
    queries = np.asarray(workload.queries)
    L, H, T, d = keys.shape
    if T == 0:
        raise ValueError("empty prefill")
    window = max(T // 8, 1)
    rows = feature_rows(T, max_rows)
    kd = torch.as_tensor(keys.reshape(L * H, T, d), dtype=torch.float64, device="cuda")
    qd = torch.as_tensor(queries.reshape(L * H, T, d)[:, rows], dtype=torch.float64, device="cuda")
    u, m = controller_stats_device(kd, qd, rows, window)
    u_hat, s_hat = normalize_features(u.cpu().numpy().reshape(L, H), m.cpu().numpy().reshape(L, H))
    r_q = float(np.mean(np.linalg.norm(queries, axis=-1)))
    return ControllerFeatures(u_hat=u_hat, s_hat=s_hat, r_q=r_q, omega=config.omega,
                              alpha_theta=config.alpha_theta, alpha_r=config.alpha_r,
                              segments=np.asarray(workload.segments), prefill=T)


def protected_mask(workload, config: ControllerConfig) -> np.ndarray:
    L, H, T, _ = np.asarray(workload.keys).shape
    mask = np.zeros((L, H, T), dtype=bool)
    for lo, hi in config.protect_spans:
        if not (0 <= lo <= hi <= T):
            raise ValueError(f"protect span {(lo, hi)} outside [0, {T}]")
        mask[:, :, lo:hi] = True
    if config.protect_outliers:
        mask |= np.asarray(workload.outliers)
    return mask
