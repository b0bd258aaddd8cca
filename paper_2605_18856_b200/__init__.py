"""B200-native Spherical KV decode hot path (arXiv 2605.18856).

Drop-in for the reference `sphkv` package's hot-path API (sphkv/__init__.py:
4-18): ADA encode/attend, RDR allocate, the paged cache object and its config
schema.  Compute runs in hand-written sm_100a kernels (libsphkv_b200.so,
C ABI in include/sphkv_b200.h); there is no CPU fallback.
"""

from . import bitpack, gate, rollout, synth
from ._lib import InfeasibleProtectionError
from .codec import (AngleCode, RadiusCode, SphericalKey, TierSpec, TierTable, angles_from_unit,
                    cos_from_angles, cos_from_codes, decode_key, encode_batch, encode_key,
                    from_spherical, quantize_angles, rate_bits, to_spherical)
from .controller import (ControllerConfig, ControllerFeatures, StateId, StateScores,
                         TierAssignment, allocate_greedy, compute_features, downtier_before_drop,
                         full_best_tier_assignment, protected_mask, score_and_best_tier,
                         score_states)
from .decode import (AttentionOutput, ada_decode, angle_logits, dense_decode, dense_logits,
                     recon_logits,
                     logit_drift_bound, lse_merge, softmax_mix, stable_softmax)
from .gate import GateConfig, GateState, danger_score, gate_step, margin
from .plan import DecodePlan, plan_dense, plan_store
from .rollout import DecodeStepper
from .store import (DenseStore, PagedStore, ResidentBreakdown, TrafficMeter, dense_mem_estimate,
                    pack_device, pack_pages_arrays)

__version__ = "0.1.0"
