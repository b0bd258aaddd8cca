"""Golden vectors for controller.compute_features, made by
running the REAL reference (read-only checkout) in the build container:
    python tests/golden/make_golden_features.py
Writes tests/golden/golden_features.npz (keys, queries, segments and the
reference's u_hat / s_hat / r_q for two seeded workloads; the second one has
more prefill rows than MAX_FEATURE_ROWS, exercising the row subsampling)."""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sphkv import controller, workload  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_features.npz")
cases = {
    "small": workload.WorkloadConfig(d=16, layers=2, heads=4, prefill=256, prefix_end=128,
                                     retrieved_end=224, seed=3),
    "rows": workload.WorkloadConfig(d=16, layers=1, heads=2, prefill=1200, prefix_end=800,
                                    retrieved_end=1000, seed=5),
}
blob = {}
for name, cfg in cases.items():
    wl = workload.generate(cfg)
    feat = controller.compute_features(wl, controller.ControllerConfig())
    blob[name + "_keys"] = wl.keys
    blob[name + "_queries"] = wl.queries
    blob[name + "_segments"] = wl.segments
    blob[name + "_u_hat"] = feat.u_hat
    blob[name + "_s_hat"] = feat.s_hat
    blob[name + "_r_q"] = np.float64(feat.r_q)
np.savez_compressed(OUT, **blob)
print("wrote", OUT, {k: v.shape for k, v in blob.items()})
