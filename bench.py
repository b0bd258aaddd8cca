"""Benchmark: ADA+RDR paged decode on B200 (BASELINE.json metric).

Default workload = config c5 (the north_star target): Llama-3.1-8B attention
geometry (32 layers, 32 Q / 8 KV heads, d = d_v = 128), one 128K-token
sequence, P = 256, panel tiers, RDR budget bisected PER SEQUENCE to a 30%
resident KV-byte reduction vs dense bf16 (ref controller.py:328-341: one
budget per store = per sequence).  A step = one decode token: one ADA decode
launch per layer (CUDA-graph captured; the split-context LSE merge is fused
into the kernel), over inputs already resident in HBM (11+ GB >> 126 MB L2,
so no flush is needed between steps).  `e2e` repeats the step through the
C-ABI call path with the step's queries copied from pinned host memory and the
attention outputs copied back, inside the timed region.

Every run checks its own workload: sampled (seq, layer, kv-head) slices are
re-encoded, packed and attended by the CPU oracle (oracle/, host numpy) and
compared with the device logits and with the outputs of the timed launches
(`parity` in the JSON line; --no-parity skips it).

Other workloads: --config c1 (one layer, 8K), c2 (B=16, 32K), c3 (Qwen2.5-14B
geometry, B=8, 128K, G=5), c4 (gpt-oss-20b geometry, sliding-window layers).
c2 and c3 do not fit next to a dense copy on one GPU: add --no-dense.

N > 1 (torchrun): `--mode split` (default for B = 1) cuts every (layer,
kv-head) page list by page range; partial softmax states are all-gathered
over NCCL and LSE-merged (strong scaling).  `--mode shard` (default for
B > 1) gives each rank whole (sequence, kv-head) page sets: no collective; a
sequence whose heads span ranks runs the same deterministic per-sequence
allocation on each of them.  `--impl reference` times the reference CPU
algorithm (the numpy oracle port, oracle/) on one host-generated slice; it
loads no product code.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (batch, layers, kv_heads, G, tokens, d, description)
    "c1": (1, 1, 8, 4, 8192, 128, "Single-layer ADA+RDR paged decode, Llama-3.1-8B head geometry, B=1, T=8K"),
    "c2": (16, 32, 8, 4, 32768, 128, "Llama-3.1-8B geometry, 32 layers, B=16, T=32K, RDR 30% KV-byte reduction"),
    "c3": (8, 48, 8, 5, 131072, 128, "Qwen2.5-14B geometry (40 Q / 8 KV heads, d=128), 48 layers, B=8, T=128K"),
    "c4": (4, 24, 8, 8, 131072, 64, "gpt-oss-20b geometry (64 Q / 8 KV heads, d=64), 24 layers "
                                   "alternating sliding-window-128 (even) / full (odd), B=4, T=128K"),
    "c5": (1, 32, 8, 4, 131072, 128, "Single 128K sequence, Llama-3.1-8B geometry, 32 layers, B=1"),
}
SWA_CONFIGS = {"c4": 128}  # sliding-window layers (even): only the last W tokens are retained
# (seq, layer, kv-head) slices checked against the CPU oracle in every run
PARITY_SLICES = {"c1": [(0, 0, 0), (0, 0, 5)], "c2": [(0, 1, 0), (5, 17, 6)],
                 "c3": [(0, 1, 0), (3, 40, 7)], "c4": [(0, 0, 3), (0, 1, 6)],
                 "c5": [(0, 1, 0), (0, 17, 5)]}
PAGE = 256
METRIC = "ADA decode tokens/s at 128K ctx, achieved HBM GB/s vs peak, KV bytes/token"
LOGIT_TOL = 1e-3
OUT_TOL = 1e-3


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def seq_seed(seed, b):
    return seed + 7919 * b


def load_traffic(cfg_name, kernel="k_ada_decode"):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture (profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum
    of one `ncu --set full` launch of this config), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t[cfg_name][kernel]
        return int(e["dram_bytes_per_launch"]), e["source"]
    except Exception:
        return None, None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    def __init__(self):
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        dev = os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or "0"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={dev}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip().splitlines()
                if out:
                    self.samples.append([x.strip() for x in out[0].split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def owned_pairs(B, H, rank, world, mode):
    """(seq, kv-head) pairs this rank decodes: all of them for the page-range
    split; a contiguous block of the b-major pair list for shard mode."""
    if mode == "split" or world == 1:
        return [(b, h) for b in range(B) for h in range(H)]
    n = B * H
    return [divmod(i, H) for i in range(rank * n // world, (rank + 1) * n // world)]


def calibrated_tiers(G, d, seed):
    """Panel tiers calibrated on a 512-key sample (cli.py:72-81 recipe) drawn
    from the workload distribution with a fixed seed, identical on every rank."""
    import torch
    from paper_2605_18856_b200 import synth

    wl = synth.generate(1, 8, 8, G, 4096, d, seed=seed + 99991)  # 64 (l, h) topics
    idx = np.random.default_rng(seed).choice(64 * 4096, size=512, replace=False)
    sample = wl.keys.view(-1, d)[torch.as_tensor(idx, device="cuda")].double().cpu().numpy()
    return synth.panel_tiers(sample_keys=sample, seed=seed)


def build_workload(cfg_name, rank=0, world=1, mode="split", seed=0, dense=True, reduction=0.30,
                   parity=True):
    """Per owned sequence: generate the synthetic KV on the device, run the
    prefill pipeline (encode radii, controller features, RDR score, budget
    bisection, greedy allocation), pack the owned groups into one shared
    store (and the dense baseline store), then free the raw K/V.  Returns a
    dict of device objects, per-sequence budget stats, setup timings and the
    host copies of the owned parity slices."""
    import torch
    import paper_2605_18856_b200 as sk
    from paper_2605_18856_b200 import _lib, synth
    from paper_2605_18856_b200.controller import allocate_greedy_device, score_states_device
    from paper_2605_18856_b200.store import code_block_bytes

    B, L, H, G, T, d, _ = CONFIGS[cfg_name]
    pairs = owned_pairs(B, H, rank, world, mode)
    heads_of = {}
    for b, h in pairs:
        heads_of.setdefault(b, []).append(h)
    tim = {"generate_s": 0.0, "encode_radii_ms": 0.0, "features_s": 0.0, "rdr_score_ms": 0.0,
           "bisection_s": 0.0, "rdr_allocate_ms": [], "pack_ms": 0.0, "dense_fill_ms": 0.0}
    t0 = time.time()
    tiers = calibrated_tiers(G, d, seed)
    tim["calibration_s"] = time.time() - t0
    tl = [(t.id, t.angle_bits, t.radius_bits, t.meta_bits) for t in tiers.tiers]
    tier_ids = torch.as_tensor([t.id for t in tiers.tiers], device="cuda")
    lut = torch.full((64,), -1, dtype=torch.int64, device="cuda")
    lut[tier_ids] = torch.arange(len(tiers.tiers), device="cuda")
    gpb = L * H  # groups per sequence
    gid = torch.arange(gpb, device="cuda").repeat_interleave(T)
    swa = SWA_CONFIGS.get(cfg_name)
    outside = None
    if swa:  # even layers: z = 0 outside the window (no sinks)
        lay = torch.arange(L, device="cuda")
        tok = torch.arange(T, device="cuda")
        outside = ((lay[:, None, None] % 2 == 0) & (tok[None, None, :] < T - swa)).expand(
            L, H, T).reshape(-1)
    dense_res_seq = synth.dense_resident_total(gpb, T, d, d, PAGE)
    st, ds = None, (sk.DenseStore(L, H, d, d, PAGE, batch=B) if dense else None)
    q_all = torch.zeros((B * gpb, G, d), dtype=torch.float32, device="cuda")
    feat_u = np.zeros(B * gpb)
    feat_s = np.zeros(B * gpb)
    feat_rq = []
    seq_info, host_slices = [], {}
    want_slices = [s for s in PARITY_SLICES.get(cfg_name, []) if (s[0], s[2]) in pairs] \
        if parity else []
    hist = np.zeros(64, dtype=np.int64)
    for b in sorted(heads_of):
        hs = sorted(heads_of[b])
        h0, h1 = hs[0], hs[-1] + 1
        t0 = time.time()
        wl = synth.generate(1, L, H, G, T, d, seed=seq_seed(seed, b))
        torch.cuda.synchronize()
        tim["generate_s"] += time.time() - t0
        n = gpb * T
        t0 = time.time()
        radii = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.check(_lib.require_gpu().sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, d,
                                                         radii.data_ptr(), _lib.stream_ptr()))
        torch.cuda.synchronize()
        tim["encode_radii_ms"] += (time.time() - t0) * 1e3
        t0 = time.time()
        u_hat, s_hat, r_q = synth.features(wl)  # normalized over this sequence's (l, h)
        torch.cuda.synchronize()
        tim["features_s"] += time.time() - t0
        feat_u[b * gpb:(b + 1) * gpb] = u_hat
        feat_s[b * gpb:(b + 1) * gpb] = s_hat
        feat_rq.append(r_q)
        seg_omega = torch.as_tensor(np.asarray(synth.PANEL_OMEGA)[wl.segments], device="cuda")
        prot = torch.zeros(n, dtype=torch.uint8, device="cuda")
        t0 = time.time()
        best, score, nu, dd = score_states_device(
            radii.view(L, H, T), torch.as_tensor(u_hat, device="cuda"),
            torch.as_tensor(s_hat, device="cuda"), seg_omega, r_q, 1.0, 1.0, tiers,
            synth.PANEL_LAMBDA, prot.view(L, H, T), d)
        torch.cuda.synchronize()
        tim["rdr_score_ms"] += (time.time() - t0) * 1e3
        del score, dd

        def windowed(z, tier):
            if outside is not None:
                z = z.masked_fill(outside.view_as(z), 0)
                tier = tier.masked_fill(outside.view_as(tier), 0)
            return z, tier

        def counts_of(tier):
            idx = gid * len(tiers.tiers) + lut[tier.view(-1).long()]
            return torch.bincount(idx, minlength=gpb * len(tiers.tiers)).view(gpb, -1).cpu().numpy()

        # per-sequence budget bisection: resident(ADA) <= (1 - R) resident(dense)
        target = (1.0 - reduction) * dense_res_seq
        dense_key_bits = n * d * 16
        lo, hi = 0.0, 1.0
        best_frac, best_asg = None, None
        t0 = time.time()
        for _ in range(14):
            mid = 0.5 * (lo + hi)
            ta = time.time()
            z, tier = allocate_greedy_device(best, nu, prot, int(mid * dense_key_bits), tiers, d)
            z, tier = windowed(z, tier)
            torch.cuda.synchronize()
            tim["rdr_allocate_ms"].append((time.time() - ta) * 1e3)
            cnt = counts_of(tier)
            res = synth.resident_total(cnt, tiers, d, d, PAGE, gpb)
            if res <= target:
                lo, best_frac, best_asg = mid, mid, (z, tier, res, cnt)
            else:
                hi = mid
        tim["bisection_s"] += time.time() - t0
        z, tier, res, cnt = best_asg
        del best, nu
        if st is None:  # pools sized from this sequence's allocation x owned sequences
            nseq = len(heads_of)
            blocks = np.array([code_block_bytes(d, PAGE, t.angle_bits, t.radius_bits)
                               if t.id else 0 for t in tiers.tiers], dtype=np.int64)
            pg = -(-cnt // PAGE)
            pages = int(pg.sum()) * nseq
            cbytes = int((pg * blocks[None, :]).sum()) * nseq
            slack = B * gpb * (len(tiers.tiers) + 2)
            st = sk.PagedStore(tiers, L, H, d, d, PAGE, batch=B, capacity_tokens=T,
                               append_tokens=256, max_pages=int(pages * 1.05) + slack,
                               code_bytes=int(cbytes * 1.05) + slack * int(blocks.max()))
        t0 = time.time()
        vals = wl.values.view(-1, d)
        keys = wl.keys.view(-1, d)
        ranges = [(0, gpb)] if (h0, h1) == (0, H) else [(l * H + h0, h1 - h0) for l in range(L)]
        for r0, rn in ranges:
            s0, s1 = r0 * T, (r0 + rn) * T
            sk.pack_device(st, keys=keys[s0:s1], radii=radii[s0:s1], values=vals[s0:s1],
                           z=z.view(-1)[s0:s1], tier=tier.view(-1)[s0:s1], protect=prot[s0:s1],
                           tokens=T, groups=(b * gpb + r0, rn))
        torch.cuda.synchronize()
        tim["pack_ms"] += (time.time() - t0) * 1e3
        if ds is not None:
            t0 = time.time()
            for r0, rn in ranges:
                ds.bulk_load(wl.keys[r0:r0 + rn], wl.values[r0:r0 + rn], groups=(b * gpb + r0, rn))
            torch.cuda.synchronize()
            tim["dense_fill_ms"] += (time.time() - t0) * 1e3
        q_all[b * gpb:(b + 1) * gpb] = wl.queries
        hist += torch.bincount(tier.view(-1).long(), minlength=64).cpu().numpy()
        seq_info.append({"seq": b, "heads": [h0, h1], "budget_frac_of_dense_key_bits": best_frac,
                         "resident_ada": int(res), "resident_dense": int(dense_res_seq),
                         "resident_ratio": res / dense_res_seq})
        for (sb, sl, sh) in want_slices:
            if sb != b:
                continue
            g = sl * H + sh
            host_slices[(sb, sl, sh)] = dict(
                keys=wl.keys[g].double().cpu().numpy(), values=wl.values[g].double().cpu().numpy(),
                q=wl.queries[g].double().cpu().numpy(),
                z=z.view(gpb, T)[g].cpu().numpy(), tier=tier.view(gpb, T)[g].cpu().numpy())
        del wl, radii, z, tier, keys, vals, prot
        torch.cuda.empty_cache()
    tim["rdr_allocate_ms"] = float(np.median(tim["rdr_allocate_ms"])) if tim["rdr_allocate_ms"] else 0.0
    info = {"tier_items": {str(t.id): int(hist[t.id]) for t in tiers.tiers},
            "per_sequence": seq_info,
            "budget": f"per sequence, {reduction:.0%} resident KV-byte reduction vs dense bf16",
            "resident_ada": sum(s["resident_ada"] for s in seq_info),
            "resident_dense": sum(s["resident_dense"] for s in seq_info)}
    info["resident_ratio"] = info["resident_ada"] / info["resident_dense"]
    return dict(st=st, ds=ds, q=q_all, tiers=tiers, tl=tl, info=info, timings=tim, pairs=pairs,
                slices=host_slices, u_hat=feat_u, s_hat=feat_s,
                r_q=float(np.mean(feat_rq)) if feat_rq else 0.0)


def time_events(fn, iters, stream):
    import torch

    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        s.record(stream)
        for _ in range(iters):
            fn()
        e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def oracle_slice(sl, tl, G, budget_s=20.0, steps=3):
    """The reference algorithm (oracle port, host numpy) on one slice: encode,
    pack, attend every query head.  Returns ([(logits, out)] per head, warm
    seconds per slice, cold seconds)."""
    from oracle import sphkv_oracle as O

    T, d = sl["keys"].shape
    r, ang = O.encode_batch(sl["keys"])
    ost = O.pack_pages(tl, sl["z"].reshape(1, 1, T), sl["tier"].reshape(1, 1, T),
                       np.zeros((1, 1, T), bool), r.reshape(1, 1, T), ang.reshape(1, 1, T, d - 1),
                       sl["values"].reshape(1, 1, T, d), PAGE)
    rq, qf = O.query_features(sl["q"])
    cache = O.FeatureCache()
    t0 = time.time()
    res = [O.head_attend(ost, 0, 0, rq[g], qf[g], cache) for g in range(G)]
    cold = time.time() - t0
    times = []
    t_end = time.time() + budget_s
    for _ in range(steps):
        t0 = time.time()
        for g in range(G):
            O.head_attend(ost, 0, 0, rq[g], qf[g], cache)
        times.append(time.time() - t0)
        if time.time() > t_end:
            break
    return res, float(np.median(times)), cold


def reference_arm(args, config, B, L, H, G, T, d):
    """--impl reference: the reference algorithm on the host only (oracle/,
    numpy, all host threads): one (layer, kv-head) slice generated, calibrated,
    scored, allocated (per-slice budget bisection), packed and attended;
    tokens/s extrapolated from the slice to all B*L*H slices of a step."""
    from oracle import sphkv_oracle as O

    t_setup = time.time()
    keys, values, q, qdraw, seg = O.generate_slice(T, d, G, seed=1234)
    tl = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 6, 8, 8), (4, 7, 8, 8), (5, 12, 14, 8),
          (6, 15, 16, 8)]  # panel tiers (pkg/configs/panel.cfg:50-56)
    eps = O.calibrate(tl, keys[np.random.default_rng(0).choice(T, 512, replace=False)], 0)
    _, _, r_q = O.features_slice(keys, qdraw)
    r, ang = O.encode_batch(keys)
    prot = np.zeros((1, 1, T), bool)
    sc = O.score_states(r.reshape(1, 1, T), np.ones((1, 1)), np.zeros((1, 1)), r_q,
                        (0.02, 2.0, 1.0), seg, 1.0, 1.0, tl, eps, 3e-5, prot, d)
    dense_res = T * 2 * d * 2 + 16 * (-(-T // PAGE)) + 30 + 8 * (1 + (-(-T // PAGE)))
    lo, hi, best = 0.0, 1.0, None
    for _ in range(12):
        mid = 0.5 * (lo + hi)
        z, tier = O.allocate_greedy(sc["best_tier"], sc["nu"], prot, int(mid * T * d * 16), tl, d)
        if O.resident_total(z[0, 0], tier[0, 0], tl, d, d, PAGE) <= 0.7 * dense_res:
            lo, best = mid, (z, tier)
        else:
            hi = mid
    z, tier = best
    sl = dict(keys=keys, values=values, q=q, z=z[0, 0], tier=tier[0, 0])
    setup = time.time() - t_setup
    samples = []
    _, t, cold = oracle_slice(sl, tl, G, steps=1)
    for _ in range(max(args.warmup - 1, 0)):
        oracle_slice(sl, tl, G, steps=1)
    for _ in range(args.steps):
        _, t, _ = oracle_slice(sl, tl, G, steps=1)
        samples.append(t)
    t_slice = float(np.median(samples))
    value = 1.0 / (t_slice * B * L * H)
    cores = os.cpu_count()
    kept = {str(t[0]): int(np.count_nonzero(tier == t[0])) for t in tl}
    sample = (f"oracle _head_attend (numpy, all host BLAS threads) for {G} q-heads of one "
              f"host-generated (layer, kv-head) slice of {T} tokens (reference workload "
              f"distribution, panel tiers calibrated on the host, features of that slice, "
              f"per-slice budget bisection to 30% resident reduction; tier items {kept}; setup "
              f"{setup:.1f} s, cold pass {cold:.2f} s); one step = one warm slice = "
              f"{t_slice * 1e3:.1f} ms, tokens/s extrapolated x{B * L * H} slices")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_slice * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="auto", choices=["auto", "split", "shard"])
    ap.add_argument("--reduction", type=float, default=0.30,
                    help="RDR budget: resident KV-byte reduction vs dense bf16, per sequence")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--profile", action="store_true", help="few steps, no graphs (for ncu)")
    ap.add_argument("--open-reserve", type=float, default=16.0,
                    help="decode steps with appends: tiles of prefill the last unit of each "
                    "group leaves for the appended pages (plan_store open_reserve_tiles)")
    ap.add_argument("--no-appends", action="store_true",
                    help="skip the full decode steps (attention + gate + append scoring + "
                         "append of one new key per group, rollout.DecodeStepper)")
    ap.add_argument("--hbyte", action="store_true",
                    help="2-bit tier through the per-query h-byte tables (csrc/hb_tile.cuh)")
    ap.add_argument("--units-per-cta", type=int, default=1)
    ap.add_argument("--tail", type=float, default=0.0,
                    help="fraction of each CTA's share cut into small dynamically claimed units")
    ap.add_argument("--unfused", action="store_true",
                    help="separate LSE-merge launch per layer (default: merge fused in the decode)")
    ap.add_argument("--dynamic", action="store_true",
                    help="CTAs claim units from a global queue (longest first)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))  # N > 1 only under torchrun
    local = int(os.environ.get("LOCAL_RANK", "0"))
    B, L, H, G, T, d, desc = CONFIGS[args.config]
    mode = args.mode if args.mode != "auto" else ("split" if B == 1 else "shard")
    if world == 1:
        mode = "single"
    config = {"workload": f"{args.config}: {desc}", "page_size": PAGE, "tiers": "panel",
              "rdr_budget": f"per sequence, {args.reduction:.0%} resident KV-byte reduction vs "
                            f"dense bf16",
              "l2": "inputs larger than L2 (no flush needed)", "batch": B, "layers": L,
              "kv_heads": H, "q_heads": H * G, "tokens": T, "d": d,
              "parallelism": {"single": "single GPU",
                              "split": f"page-range split x{world} + NCCL all-gather LSE merge",
                              "shard": f"batch x KV-head shards x{world}, no collective"}[mode],
              "launch": "one decode launch per layer, split merge fused in-kernel (CUDA graph)"}

    import torch

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, config, B, L, H, G, T, d)
        return

    # SPHKV_BENCH_GLOO=1 (debug of the N > 1 path on a single GPU): every rank
    # on cuda:0, gloo process group, the all-gather staged through host memory
    gloo_dbg = world > 1 and os.environ.get("SPHKV_BENCH_GLOO") == "1"
    if gloo_dbg:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if gloo_dbg:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2605_18856_b200 as sk
    from paper_2605_18856_b200 import _lib, plan as planmod

    W = build_workload(args.config, rank, world, "split" if mode == "single" else mode,
                       dense=not args.no_dense, reduction=args.reduction,
                       parity=not args.no_parity and rank == 0)
    st, ds, q = W["st"], W["ds"], W["q"]
    st.hbyte_tables = args.hbyte
    pairs = set(W["pairs"])
    log("setup", json.dumps(W["timings"]), json.dumps(W["info"]))

    layer_groups = [[(b * L + l) * H + h for b in range(B) for h in range(H) if (b, h) in pairs]
                    for l in range(L)]

    def ada_plan(groups):
        if mode == "split":
            return planmod.plan_store_range(st, groups, rank, world, units_per_cta=args.units_per_cta)
        return planmod.plan_store(st, groups=groups, units_per_cta=args.units_per_cta,
                                  dynamic=args.dynamic, tail=args.tail)

    plans = [ada_plan(g) for g in layer_groups]
    n_launch = len(plans)
    swa = SWA_CONFIGS.get(args.config)
    npg = -(-T // PAGE)
    win = [(T - swa) if swa and l % 2 == 0 else 0 for l in range(L)]  # first attended token
    dplans = [planmod.plan_dense(ds, groups=layer_groups[l], dynamic=args.dynamic,
                                 pages=(win[l] // PAGE, npg))
              for l in range(L)] if ds is not None and mode != "split" else []
    if swa:
        config["sliding_window"] = (f"{swa} tokens on even layers (ADA: z = 0 outside the window; "
                                    f"dense baseline: the same last {swa} tokens)")
    outs = [torch.empty((len(p.group_ids) * G, d), dtype=torch.float32, device="cuda") for p in plans]
    parts = [sk.decode._partials(p, G, d) for p in plans]
    lib = _lib.lib()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    fused = mode != "split" and not args.unfused

    def decode_layers(with_merge=True):
        for l, p in enumerate(plans):
            if fused:
                _lib.check(lib.sphkv_ada_decode_fused(
                    st.cptr_for(G), q.data_ptr(), G, p.units.data_ptr(), p.n_units, parts[l].data_ptr(),
                    p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids),
                    p.ctl.data_ptr(), outs[l].data_ptr(), int(p.dynamic), p.grid, sp))
                continue
            _lib.check(lib.sphkv_ada_decode(st.cptr_for(G), q.data_ptr(), G, p.units.data_ptr(),
                                            p.n_units, parts[l].data_ptr(), None, None, p.grid, sp))
            if with_merge and mode != "split":
                _lib.check(lib.sphkv_lse_merge(parts[l].data_ptr(), p.slot_begin.data_ptr(),
                                               len(p.group_ids), G, d, outs[l].data_ptr(), sp))

    dparts = [sk.decode._partials(p, G, d) for p in dplans]
    douts = [torch.empty((len(p.group_ids) * G, d), dtype=torch.float32, device="cuda") for p in dplans]

    def dense_layers():
        for l, p in enumerate(dplans):
            _lib.check(lib.sphkv_dense_decode_window(
                ds.cptr, q.data_ptr(), G, p.units.data_ptr(), p.n_units, dparts[l].data_ptr(),
                p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids),
                p.ctl.data_ptr(), douts[l].data_ptr(), int(p.dynamic), win[l], p.grid, sp))

    if args.profile:
        with torch.cuda.stream(stream):
            for _ in range(max(args.steps, 1)):
                decode_layers()
                if dplans:
                    dense_layers()
        torch.cuda.synchronize()
        log("profile run done")
        return

    step_fn = decode_layers
    out_all = None
    if mode == "split":
        # page-range split of every (seq, layer, kv-head) list: per layer the
        # local splits are LSE-merged into one partial state per (group, q-head);
        # the states of all layers go out in ONE all-gather per step (valid in
        # this attention-only benchmark, where every layer's query is given),
        # then one merge over ranks yields every layer's output on every rank.
        import torch.distributed as dist

        ng = len(plans[0].group_ids)
        F = G * (d + 2)
        state = torch.empty((n_launch, ng, F), dtype=torch.float32, device="cuda")
        gathered = torch.empty((world, n_launch, ng, F), dtype=torch.float32, device="cuda")
        out_all = torch.empty((n_launch * ng * G, d), dtype=torch.float32, device="cuda")

        def local_layers():  # each rank's share: one fused launch per layer -> states
            for l, p in enumerate(plans):
                _lib.check(lib.sphkv_ada_decode_state(
                    st.cptr_for(G), q.data_ptr(), G, p.units.data_ptr(), p.n_units,
                    parts[l].data_ptr(), p.slot_group.data_ptr(), p.slot_begin.data_ptr(), ng,
                    p.ctl.data_ptr(), state[l].data_ptr(), p.grid, sp))

        with torch.cuda.stream(stream):
            for _ in range(2):
                local_layers()
        torch.cuda.synchronize()
        lgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(lgraph, stream=stream):
            local_layers()

        def step_fn():
            with torch.cuda.stream(stream):
                lgraph.replay()
            with torch.cuda.stream(stream):
                if gloo_dbg:
                    g_h = torch.empty(gathered.numel(), dtype=torch.float32)
                    dist.all_gather_into_tensor(g_h, state.view(-1).cpu())
                    gathered.view(-1).copy_(g_h)
                else:
                    dist.all_gather_into_tensor(gathered.view(-1), state.view(-1))
            planmod.merge_gathered(n_launch * ng, world, gathered, G, d, out_all, stream)

    # warmup + graph capture of the step (launch-bound loop of per-layer kernels)
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step_fn()
    torch.cuda.synchronize()
    if mode != "split":
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step_fn()
        run = graph.replay
    else:
        run = step_fn

    clocks = ClockSampler()
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for _ in range(args.steps):
            run()
        ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device="cpu" if gloo_dbg else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tokens_per_s = B / (ms * 1e-3)

    # parity of this run's own workload: oracle on the host vs the device
    # logits (debug launch on the same pages) and the timed launches' outputs
    parity = None
    cpu = None
    if W["slices"]:
        worst_lg = worst_out = 0.0
        checked = []
        first_t = None
        for (b, l, h), sl in W["slices"].items():
            res, t_warm, cold = oracle_slice(sl, W["tl"], G)
            if first_t is None:
                first_t, first_cold = t_warm, cold
            lg, _ = sk.decode.attend_heads(st, l, h, sl["q"], seq=b)
            g = (b * L + l) * H + h
            if mode == "split":
                ng = len(plans[0].group_ids)
                pos = list(plans[l].group_ids).index(g)
                got = out_all[(l * ng + pos) * G:(l * ng + pos + 1) * G].double().cpu().numpy()
            else:
                pos = list(plans[l].group_ids).index(g)
                got = outs[l][pos * G:(pos + 1) * G].double().cpu().numpy()
            for gi in range(G):
                want_lg, want_out = res[gi]
                if want_lg.size:
                    e = float(np.max(np.abs(lg[gi] - want_lg) / np.maximum(1.0, np.abs(want_lg))))
                    worst_lg = max(worst_lg, e)
                den = max(float(np.max(np.abs(want_out))), 1e-30)
                worst_out = max(worst_out, float(np.max(np.abs(got[gi] - want_out))) / den)
            checked.append({"seq": b, "layer": l, "kv_head": h, "items": int(lg.shape[1])})
        parity = {"max_logit_rel": worst_lg, "max_out_rel": worst_out, "slices": checked,
                  "tol": {"logit": LOGIT_TOL, "out": OUT_TOL},
                  "ok": worst_lg <= LOGIT_TOL and worst_out <= OUT_TOL,
                  "oracle": "oracle/sphkv_oracle.py: host encode + pack + head_attend of the "
                            "slice's keys/values/queries (fp64); device logits from a debug "
                            "launch on the bench's own pages, outputs from the timed launches"}
        log("parity", json.dumps(parity))
        if world == 1 and not args.no_cpu:
            cpu = {"value": 1.0 / (first_t * B * L * H), "unit": "tokens/s",
                   "cores": os.cpu_count(), "kind": "port",
                   "sample": f"oracle _head_attend (numpy, all BLAS threads) on the first parity "
                             f"slice x {G} q-heads of this workload (warm page caches; cold "
                             f"{first_cold:.2f} s), scaled by {B * L * H} slices"}

    # kernel-level timing of the dominant kernel (ADA decode, all layers)
    dec_ms = time_events(lambda: decode_layers(with_merge=False), max(args.steps // 2, 3),
                         stream) / n_launch
    # (fused: the per-launch time includes the in-kernel split merge)
    bytes_total = st.stream_bytes_total()  # owned groups' pages (algorithmic, store.py:315-322)
    if mode == "split":
        bytes_total = bytes_total // world
    qbytes = sum(len(p.group_ids) for p in plans) * G * d * 4
    part_bytes = sum(p.n_slots for p in plans) * G * (d + 2) * 4
    alg_bytes_per_launch = (bytes_total + qbytes + part_bytes) / n_launch
    peak, peak_kind = load_peaks()
    traffic, traffic_src = load_traffic(args.config) if world == 1 else (None, None)
    achieved = alg_bytes_per_launch / (dec_ms * 1e-3) / 1e9
    seqs_owned = len(pairs) / H  # sequence equivalents decoded on this rank
    kv_bytes_token = W["info"]["resident_ada"] / (T * seqs_owned)
    dense_stream_bytes = sum(
        len(layer_groups[l]) * (16 * (npg - win[l] // PAGE) + (T - win[l]) * 2 * d * 2)
        for l in range(L))

    # dense baseline (same scheduler, page size, bf16 K / fp16 V, same windows)
    dense = None
    if dplans:
        with torch.cuda.stream(stream):
            for _ in range(3):
                dense_layers()
        dgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(dgraph, stream=stream):
            dense_layers()
        dms = time_events(dgraph.replay, args.steps, stream)
        if world > 1:
            t = torch.tensor([dms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dms = float(t.item())
        dbytes = dense_stream_bytes + qbytes
        dense = {"value": B / (dms * 1e-3), "unit": "tokens/s", "ms_per_step": dms,
                 "achieved_gbs": dbytes / (dms * 1e-3) / 1e9,
                 "frac_of_peak": dbytes / (dms * 1e-3) / 1e9 / peak,
                 "stream_bytes_per_step": int(dbytes),
                 "kv_bytes_per_token": W["info"]["resident_dense"] / (T * seqs_owned)}

    # e2e: host q (pinned) -> device, step, outputs -> host (pinned), per step
    qh = q.cpu().pin_memory()
    res_dev = out_all if out_all is not None else None
    n_out = res_dev.shape[0] if res_dev is not None else sum(o.shape[0] for o in outs)
    oh = torch.empty((n_out, d), dtype=torch.float32).pin_memory()
    ocat = torch.empty_like(oh, device="cuda")

    def e2e_step():
        q.copy_(qh, non_blocking=True)
        run()
        if res_dev is not None:
            oh.copy_(res_dev, non_blocking=True)
        else:
            torch.cat(outs, out=ocat)
            oh.copy_(ocat, non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(2):
            e2e_step()
    torch.cuda.synchronize()
    e2e_ms = time_events(e2e_step, args.steps, stream)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cpu" if gloo_dbg else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # full decode steps with appends (decode.py:415-498): the store grows by
    # one key per group per step, so this runs last
    step_app = None
    if not args.no_appends and not args.profile and mode in ("single", "shard"):
        from paper_2605_18856_b200 import synth as synthm
        from paper_2605_18856_b200.gate import GateConfig

        nsteps = args.steps
        gen = torch.Generator(device="cuda")
        gen.manual_seed(4242)
        groups = st.groups
        kn = torch.randn((nsteps + 3, groups, d), generator=gen, device="cuda") / d ** 0.5
        kn = (kn + torch.nn.functional.normalize(
            torch.randn((groups, d), generator=gen, device="cuda"), dim=-1)) * 1.0
        vn = torch.randn((nsteps + 3, groups, d), generator=gen, device="cuda").half()
        stp = sk.DecodeStepper(st, G, W["u_hat"], W["s_hat"], W["r_q"], lam=synthm.PANEL_LAMBDA,
                               omega=synthm.PANEL_OMEGA[2], gate_cfg=GateConfig(0.05, 0.5),
                               open_reserve_tiles=args.open_reserve)
        stp.capture(stream)
        for t in range(3):
            stp.step(q, kn[t], vn[t], T + t)
        torch.cuda.synchronize()

        def app_step(t):
            stp.step(None, kn[t], vn[t], T + t)

        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a0.record(stream)
            for t in range(nsteps):
                app_step(3 + t)
            a1.record(stream)
        torch.cuda.synchronize()
        app_ms = a0.elapsed_time(a1) / nsteps
        stp.finish()
        step_app = {"value": B / (app_ms * 1e-3), "unit": "tokens/s", "ms_per_step": app_ms,
                    "steps": nsteps, "what": "per step: live ADA decode of every layer with "
                    "gate margins, the decode-time gate + best-tier scoring of one new key per "
                    "(seq, layer, kv-head), and its append (one CUDA graph)",
                    "protected_heads_last_step": int((stp.mode == 2).sum())}
        if world > 1:
            t = torch.tensor([app_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            step_app["ms_per_step"] = float(t.item())
            step_app["value"] = B / (step_app["ms_per_step"] * 1e-3)

    if rank == 0:
        ada_stream_tok = (bytes_total * (world if mode == "split" else 1)) / seqs_owned
        line = {"metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True,
                "scaling": "strong" if mode in ("single", "split") else "weak",
                "vs_baseline": None, "dtype": "f32 (fp16 V, angle codes)", "data": "synthetic",
                "config": config,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "traffic_source": traffic_src,
                             "kernel": "k_ada_decode", "kernel_ms_per_launch": dec_ms,
                             "alg_bytes_per_launch": int(alg_bytes_per_launch),
                             "peak_kind": peak_kind},
                "kv_bytes_per_token": kv_bytes_token,
                "stream_bytes_per_token": ada_stream_tok,
                "resident_ratio_vs_dense": W["info"]["resident_ratio"],
                "streamed_ratio_vs_dense": (bytes_total / dense_stream_bytes
                                            if mode != "split" else None),
                "dense_baseline": dense,
                "speedup_vs_dense": (tokens_per_s / dense["value"]) if dense else None,
                "parity": parity,
                "cpu_baseline": cpu,
                "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "tokens/s",
                        "h2d_bytes_per_step": int(qh.numel() * 4),
                        "d2h_bytes_per_step": int(oh.numel() * 4)},
                "gpu_launches": args.steps * (n_launch if fused else 2 * n_launch if mode != "split"
                                              else n_launch + 1),
                "decode_step_with_appends": step_app,
                "clocks": clk, "prefill": W["timings"], "budget": W["info"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
