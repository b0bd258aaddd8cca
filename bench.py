"""Benchmark: ADA+RDR paged decode on B200 (BASELINE.json metric).

Default workload = config 5 (the north_star target): Llama-3.1-8B attention
geometry (32 layers, 32 Q / 8 KV heads, d = d_v = 128), one 128K-token
sequence, P = 256, panel tiers, RDR budget bisected to a 30% resident KV-byte
reduction vs dense bf16.  A step = one decode token: one ADA decode launch per
layer (32, CUDA-graph captured; the split-context LSE merge is fused into the
kernel), over inputs already resident in HBM (11+ GB >> 126 MB L2, so no
flush is needed between steps).  `e2e` repeats the step through the C-ABI
call path with the step's queries copied from pinned host memory and the
attention outputs copied back, inside the timed region.  Other workloads:
--config c1 (one layer, 8K), c2 (B=16, 32K; add --no-dense, the dense copy
does not fit next to it), c4 (gpt-oss-20b geometry, sliding-window layers).

N > 1 (torchrun): the sequence's page lists are split by page range across
ranks; partial softmax states are all-gathered over NCCL and LSE-merged on
every rank (strong scaling).  `--impl reference` times the reference CPU
algorithm (the numpy oracle port, oracle/) on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
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
    "c4": (4, 24, 8, 8, 131072, 64, "gpt-oss-20b geometry (64 Q / 8 KV heads, d=64), 24 layers "
                                   "alternating sliding-window-128 (even) / full (odd), B=4, T=128K"),
    "c5": (1, 32, 8, 4, 131072, 128, "Single 128K sequence, Llama-3.1-8B geometry, 32 layers, B=1"),
}
SWA_CONFIGS = {"c4": 128}  # sliding-window layers (even): only the last W tokens are retained
PAGE = 256
REDUCTION = 0.30


def log(*a):
    print(*a, file=sys.stderr, flush=True)


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


def build_workload(cfg_name, rank=0, seed=0, dense=True):
    """Generate the synthetic KV, run the device prefill pipeline (encode radii,
    RDR score, budget bisection, greedy allocation, page packing) and the dense
    baseline store.  Returns a dict of device objects + setup timings."""
    import torch
    import paper_2605_18856_b200 as sk
    from paper_2605_18856_b200 import _lib, synth
    from paper_2605_18856_b200.controller import allocate_greedy_device, score_states_device

    B, L, H, G, T, d, _ = CONFIGS[cfg_name]
    t0 = time.time()
    wl = synth.generate(B, L, H, G, T, d, seed=seed)
    torch.cuda.synchronize()
    tim = {"generate_s": time.time() - t0}
    groups = wl.groups
    n = groups * T
    # K1 pass 1: radii (fp64, numpy pairwise order)
    t0 = time.time()
    radii = torch.empty(n, dtype=torch.float64, device="cuda")
    l = _lib.require_gpu()
    _lib.check(l.sphkv_encode_radii(wl.keys.data_ptr(), _lib.BF16, n, d, radii.data_ptr(),
                                    _lib.stream_ptr()))
    torch.cuda.synchronize()
    tim["encode_radii_ms"] = (time.time() - t0) * 1e3
    # controller features + calibration (input contract, 8(d))
    t0 = time.time()
    u_hat, s_hat, r_q = synth.features(wl)
    rng = np.random.default_rng(seed)
    sample_idx = rng.choice(n, size=512, replace=False)
    sample = wl.keys.view(-1, d)[torch.as_tensor(sample_idx, device="cuda")].double().cpu().numpy()
    tiers = synth.panel_tiers(sample_keys=sample, seed=seed)
    torch.cuda.synchronize()
    tim["features_calibration_s"] = time.time() - t0
    seg_omega = torch.as_tensor(np.asarray(synth.PANEL_OMEGA)[wl.segments], device="cuda")
    prot = torch.zeros(n, dtype=torch.uint8, device="cuda")
    t0 = time.time()
    best, score, nu, dd = score_states_device(
        radii.view(B * L, H, T), torch.as_tensor(u_hat, device="cuda"),
        torch.as_tensor(s_hat, device="cuda"), seg_omega, r_q, 1.0, 1.0, tiers,
        synth.PANEL_LAMBDA, prot.view(B * L, H, T), d)
    torch.cuda.synchronize()
    tim["rdr_score_ms"] = (time.time() - t0) * 1e3
    del score, dd
    # budget bisection: resident(ADA) <= (1 - REDUCTION) * resident(dense)
    dense_res = synth.dense_resident_total(groups, T, d, d, PAGE)
    target = (1.0 - REDUCTION) * dense_res
    tier_ids = torch.as_tensor([t.id for t in tiers.tiers], device="cuda")
    lut = torch.full((64,), -1, dtype=torch.int64, device="cuda")
    lut[tier_ids] = torch.arange(len(tiers.tiers), device="cuda")
    gid = torch.arange(groups, device="cuda").repeat_interleave(T)

    swa = SWA_CONFIGS.get(cfg_name)
    if swa:  # even layers: z = 0 outside the window (no sinks)
        lay = torch.arange(B * L, device="cuda") % L
        tok = torch.arange(T, device="cuda")
        outside = ((lay[:, None, None] % 2 == 0) & (tok[None, None, :] < T - swa)).expand(
            B * L, H, T).reshape(-1)

    def windowed(z, tier):
        if swa:
            z = z.masked_fill(outside.view_as(z), 0)
            tier = tier.masked_fill(outside.view_as(tier), 0)
        return z, tier

    def resident_of(tier):
        idx = gid * len(tiers.tiers) + lut[tier.view(-1).long()]
        counts = torch.bincount(idx, minlength=groups * len(tiers.tiers)).view(groups, -1)
        return synth.resident_total(counts.cpu().numpy(), tiers, d, d, PAGE, groups)

    dense_key_bits = n * d * 16
    lo, hi = 0.0, 1.0
    best_frac, best_asg = None, None
    t0 = time.time()
    alloc_ms = []
    for _ in range(14):
        mid = 0.5 * (lo + hi)
        ta = time.time()
        z, tier = allocate_greedy_device(best, nu, prot, int(mid * dense_key_bits), tiers, d)
        z, tier = windowed(z, tier)
        torch.cuda.synchronize()
        alloc_ms.append((time.time() - ta) * 1e3)
        res = resident_of(tier)
        if res <= target:
            lo, best_frac, best_asg = mid, mid, (z, tier, res)
        else:
            hi = mid
    tim["bisection_s"] = time.time() - t0
    tim["rdr_allocate_ms"] = float(np.median(alloc_ms))
    z, tier, res = best_asg
    # K1 pass 2 + K2/K3/K6: encode + quantize + pack
    t0 = time.time()
    st = sk.PagedStore(tiers, L, H, d, d, PAGE, batch=B, capacity_tokens=T, append_tokens=256)
    sk.pack_device(st, keys=wl.keys.view(-1, d), radii=radii, values=wl.values.view(-1, d),
                   z=z.view(-1), tier=tier.view(-1), protect=prot, tokens=T)
    torch.cuda.synchronize()
    tim["pack_ms"] = (time.time() - t0) * 1e3
    del best, nu
    ds = None
    if dense:  # (c2 does not fit next to the dense copy: run it with --no-dense)
        t0 = time.time()
        ds = sk.DenseStore(L, H, d, d, PAGE, batch=B)
        ds.bulk_load(wl.keys, wl.values)
        torch.cuda.synchronize()
        tim["dense_fill_ms"] = (time.time() - t0) * 1e3
    hist = torch.bincount(tier.view(-1).long(), minlength=8).cpu().tolist()
    info = {"tier_items": {str(t.id): int(hist[t.id]) for t in tiers.tiers},
            "budget_frac_of_dense_key_bits": best_frac, "resident_ada": int(res),
            "resident_dense": int(dense_res), "resident_ratio": res / dense_res}
    return dict(wl=wl, st=st, ds=ds, tiers=tiers, radii=radii, z=z, tier=tier, info=info,
                timings=tim, u_hat=u_hat, s_hat=s_hat, r_q=r_q)


def layer_plans(st, L, H, B, rank, world, plan_fn):
    """One plan per layer (groups of that layer across the batch)."""
    plans = []
    for l in range(L):
        groups = [(b * L + l) * H + h for b in range(B) for h in range(H)]
        plans.append(plan_fn(st, groups))
    return plans


def time_events(fn, iters):
    import torch

    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def cpu_oracle_sample(W, rank, steps=3, budget_s=20.0):
    """The reference algorithm (oracle port) timed on host cores on one (layer,
    kv-head) slice of the same workload: warm _head_attend for its G query heads."""
    import torch
    from oracle import sphkv_oracle as O

    wl, z, tier = W["wl"], W["z"], W["tier"]
    T, d, G = wl.tokens, wl.d, wl.G
    g = wl.heads if wl.layers > 1 else 0  # layer 1, head 0 (full attention when layers alternate)
    keys = wl.keys[g].double().cpu().numpy()
    vals = wl.values[g].double().cpu().numpy()
    r, ang = O.encode_batch(keys)
    tl = [(t.id, t.angle_bits, t.radius_bits, t.meta_bits) for t in W["tiers"].tiers]
    zz = z.view(-1)[g * T:(g + 1) * T].cpu().numpy().reshape(1, 1, T)
    tt = tier.view(-1)[g * T:(g + 1) * T].cpu().numpy().reshape(1, 1, T)
    ost = O.pack_pages(tl, zz, tt, np.zeros((1, 1, T), bool), r.reshape(1, 1, T),
                       ang.reshape(1, 1, T, d - 1), vals.reshape(1, 1, T, d), PAGE)
    q = wl.queries[g].double().cpu().numpy()
    rq, qf = O.query_features(q)
    cache = O.FeatureCache()
    t0 = time.time()
    for gi in range(G):
        O.head_attend(ost, 0, 0, rq[gi], qf[gi], cache)  # cold: builds the page caches
    cold = time.time() - t0
    times = []
    t_end = time.time() + budget_s
    for _ in range(steps):
        t0 = time.time()
        for gi in range(G):
            O.head_attend(ost, 0, 0, rq[gi], qf[gi], cache)
        times.append(time.time() - t0)
        if time.time() > t_end:
            break
    return float(np.median(times)), cold


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--profile", action="store_true", help="few steps, no graphs (for ncu)")
    ap.add_argument("--units-per-cta", type=int, default=1)
    ap.add_argument("--tail", type=float, default=0.0,
                    help="fraction of each CTA's share cut into small dynamically claimed units")
    ap.add_argument("--unfused", action="store_true",
                    help="separate LSE-merge launch per layer (default: merge fused in the decode)")
    ap.add_argument("--dynamic", action="store_true",
                    help="CTAs claim units from a global queue (longest first)")
    ap.add_argument("--fuse-layers", action="store_true",
                    help="one decode launch over all layers (attention-only benchmark shortcut)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))  # N > 1 only under torchrun
    local = int(os.environ.get("LOCAL_RANK", "0"))
    B, L, H, G, T, d, desc = CONFIGS[args.config]
    metric = "ADA decode tokens/s at 128K ctx, achieved HBM GB/s vs peak, KV bytes/token"
    config = {"workload": f"{args.config}: {desc}", "page_size": PAGE, "tiers": "panel",
              "rdr_budget": "30% resident KV-byte reduction vs dense bf16",
              "l2": "inputs larger than L2 (no flush needed)", "batch": B, "layers": L,
              "kv_heads": H, "q_heads": H * G, "tokens": T, "d": d,
              "parallelism": f"page-range split x{world}" if world > 1 else "single GPU",
              "launch": "one decode launch per layer, split merge fused in-kernel (CUDA graph)"}

    import torch

    if args.impl == "reference":
        if rank != 0:
            return
        torch.cuda.set_device(local)
        W = build_workload(args.config, rank, dense=False)
        samples = []
        for _ in range(args.warmup):
            cpu_oracle_sample(W, rank, steps=1, budget_s=60)
        for _ in range(args.steps):
            t, _ = cpu_oracle_sample(W, rank, steps=1, budget_s=60)
            samples.append(t)
        t_slice = float(np.median(samples))
        per_token = t_slice * B * L * H  # every (seq, layer, kv head) slice costs the same
        value = 1.0 / per_token
        cores = os.cpu_count()
        line = {"impl": "reference", "metric": metric, "value": value, "unit": "tokens/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": per_token * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config,
                "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores,
                                 "kind": "port",
                                 "sample": f"oracle _head_attend, 1 (layer, kv-head) slice x {G} "
                                           f"q-heads of the {args.config} workload, scaled by "
                                           f"{B * L * H} slices"},
                "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
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

    W = build_workload(args.config, rank, dense=not args.no_dense)
    st, ds, wl = W["st"], W["ds"], W["wl"]
    log("setup", json.dumps(W["timings"]), json.dumps(W["info"]))

    def ada_plan(s, groups):
        if world == 1:
            return planmod.plan_store(s, groups=groups, units_per_cta=args.units_per_cta,
                                      dynamic=args.dynamic, tail=args.tail)
        return planmod.plan_store_range(s, groups, rank, world, units_per_cta=args.units_per_cta)

    if args.fuse_layers:
        plans = [ada_plan(st, list(range(B * L * H)))]
        config["launch"] = "one decode+merge over all layers (CUDA graph)"
    else:
        plans = layer_plans(st, L, H, B, rank, world, ada_plan)
    n_launch = len(plans)
    swa = SWA_CONFIGS.get(args.config)
    dplans = [planmod.plan_dense(ds, groups=[(b * L + l) * H + h for b in range(B) for h in range(H)],
                                 dynamic=args.dynamic,
                                 pages=(ds.n_pages_per_group - (-(-swa // PAGE)), ds.n_pages_per_group)
                                 if swa and l % 2 == 0 else None)
              for l in range(L)] if not args.no_dense else []
    if swa:
        config["sliding_window"] = (f"{swa} tokens on even layers (ADA: z = 0 outside the window; "
                                    f"dense baseline: the window's last {PAGE}-token page)")
    q = wl.queries
    outs = [torch.empty((len(p.group_ids) * G, d), dtype=torch.float32, device="cuda") for p in plans]
    parts = [sk.decode._partials(p, G, d) for p in plans]
    lib = _lib.lib()
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream

    fused = world == 1 and not args.unfused

    def decode_layers(with_merge=True):
        for l, p in enumerate(plans):
            if fused:
                _lib.check(lib.sphkv_ada_decode_fused(
                    st.cptr, q.data_ptr(), G, p.units.data_ptr(), p.n_units, parts[l].data_ptr(),
                    p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids),
                    p.ctl.data_ptr(), outs[l].data_ptr(), int(p.dynamic), p.grid, sp))
                continue
            _lib.check(lib.sphkv_ada_decode(st.cptr, q.data_ptr(), G, p.units.data_ptr(),
                                            p.n_units, parts[l].data_ptr(), None, None, p.grid, sp))
            if with_merge and world == 1:
                _lib.check(lib.sphkv_lse_merge(parts[l].data_ptr(), p.slot_begin.data_ptr(),
                                               len(p.group_ids), G, d, outs[l].data_ptr(), sp))

    def merge_layers():
        for l, p in enumerate(plans):
            _lib.check(lib.sphkv_lse_merge(parts[l].data_ptr(), p.slot_begin.data_ptr(),
                                           len(p.group_ids), G, d, outs[l].data_ptr(), sp))

    dparts = [sk.decode._partials(p, G, d) for p in dplans]
    douts = [torch.empty((len(p.group_ids) * G, d), dtype=torch.float32, device="cuda") for p in dplans]

    def dense_layers():
        for l, p in enumerate(dplans):
            if fused:
                _lib.check(lib.sphkv_dense_decode_fused(
                    ds.cptr, q.data_ptr(), G, p.units.data_ptr(), p.n_units, dparts[l].data_ptr(),
                    p.slot_group.data_ptr(), p.slot_begin.data_ptr(), len(p.group_ids),
                    p.ctl.data_ptr(), douts[l].data_ptr(), int(p.dynamic), p.grid, sp))
                continue
            _lib.check(lib.sphkv_dense_decode(ds.cptr, q.data_ptr(), G, p.units.data_ptr(),
                                              p.n_units, dparts[l].data_ptr(), p.grid, sp))
            _lib.check(lib.sphkv_lse_merge(dparts[l].data_ptr(), p.slot_begin.data_ptr(),
                                           len(p.group_ids), G, d, douts[l].data_ptr(), sp))

    if args.profile:
        with torch.cuda.stream(stream):
            for _ in range(max(args.steps, 1)):
                decode_layers()
                if not args.no_dense:
                    dense_layers()
        torch.cuda.synchronize()
        log("profile run done")
        return

    step_fn = decode_layers
    if world > 1:
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

        def step_fn():
            decode_layers(with_merge=False)
            for l, p in enumerate(plans):
                planmod.merge_local_state(p, parts[l], G, d, state[l], stream)
            with torch.cuda.stream(stream):
                if gloo_dbg:
                    g_h = torch.empty(gathered.numel(), dtype=torch.float32)
                    dist.all_gather_into_tensor(g_h, state.view(-1).cpu())
                    gathered.view(-1).copy_(g_h)
                else:
                    dist.all_gather_into_tensor(gathered.view(-1), state.view(-1))
            planmod.merge_gathered(n_launch * ng, world, gathered, G, d, out_all, stream)

    # warmup + graph capture of the step (launch-bound loop of 64 kernels)
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            step_fn()
    torch.cuda.synchronize()
    graph = None
    if world == 1:
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
    if gloo_dbg and rank == 0:  # the split + two-level merge == the single-rank decode
        ng = len(plans[0].group_ids)
        worst = 0.0
        for l in range(L):
            grp = [(b * L + l) * H + h for b in range(B) for h in range(H)]
            ref = sk.ada_decode(st, q, planmod.plan_store(st, groups=grp, units_per_cta=1))
            got = out_all[l * ng * G:(l + 1) * ng * G]
            worst = max(worst, float((got - ref).abs().max() / ref.abs().max().clamp_min(1e-30)))
        log(f"N>1 debug: max relative |split merge - single pass| over {L} layers = {worst:.3e}")

    # kernel-level timing of the dominant kernel (ADA decode, all layers)
    with torch.cuda.stream(stream):
        dec_ms = time_events(lambda: decode_layers(with_merge=False), max(args.steps // 2, 3)) / n_launch
        # (fused: the per-launch time includes the in-kernel split merge)
    bytes_total = st.stream_bytes_total()
    qbytes = B * L * H * G * d * 4
    part_bytes = sum(p.n_slots for p in plans) * G * (d + 2) * 4
    if world > 1:
        bytes_total = bytes_total // world
    alg_bytes_per_launch = (bytes_total + qbytes + part_bytes) / n_launch
    peak, peak_kind = load_peaks()
    traffic, traffic_src = load_traffic(args.config) if world == 1 else (None, None)
    achieved = alg_bytes_per_launch / (dec_ms * 1e-3) / 1e9
    kv_bytes_token = W["info"]["resident_ada"] / T

    # dense baseline (same scheduler, page size, bf16 K / fp16 V)
    dense = None
    if not args.no_dense and world == 1:
        with torch.cuda.stream(stream):
            for _ in range(3):
                dense_layers()
        dgraph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(dgraph, stream=stream):
            dense_layers()
        with torch.cuda.stream(stream):
            dms = time_events(dgraph.replay, args.steps)
        dbytes = ds.stream_bytes_total() + qbytes
        dense = {"value": B / (dms * 1e-3), "unit": "tokens/s", "ms_per_step": dms,
                 "achieved_gbs": dbytes / (dms * 1e-3) / 1e9,
                 "frac_of_peak": dbytes / (dms * 1e-3) / 1e9 / peak,
                 "stream_bytes_per_step": int(dbytes),
                 "kv_bytes_per_token": W["info"]["resident_dense"] / T}

    # e2e: host q (pinned) -> device, step, outputs -> host (pinned), per step
    qh = q.cpu().pin_memory()
    oh = torch.empty((sum(o.shape[0] for o in outs), d), dtype=torch.float32).pin_memory()
    ocat = torch.empty_like(oh, device="cuda")

    def e2e_step():
        q.copy_(qh, non_blocking=True)
        run()
        if world > 1:
            oh.copy_(out_all, non_blocking=True)
        else:
            torch.cat(outs, out=ocat)
            oh.copy_(ocat, non_blocking=True)

    with torch.cuda.stream(stream):
        for _ in range(2):
            e2e_step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t_slice, cold = cpu_oracle_sample(W, rank)
        per_token = t_slice * B * L * H
        cpu = {"value": 1.0 / per_token, "unit": "tokens/s", "cores": os.cpu_count(),
               "kind": "port",
               "sample": f"oracle _head_attend (numpy, all BLAS threads) on 1 (layer, kv-head) "
                         f"slice x {G} q-heads of this workload (warm page caches; cold "
                         f"{cold:.2f} s), scaled by {B * L * H} slices"}

    if rank == 0:
        line = {"metric": metric, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32 (fp16 V, angle codes)", "data": "synthetic", "config": config,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "traffic_source": traffic_src,
                             "kernel": "k_ada_decode", "kernel_ms_per_launch": dec_ms,
                             "alg_bytes_per_launch": int(alg_bytes_per_launch),
                             "peak_kind": peak_kind},
                "kv_bytes_per_token": kv_bytes_token,
                "stream_bytes_per_token": bytes_total + qbytes,
                "resident_ratio_vs_dense": W["info"]["resident_ratio"],
                "dense_baseline": dense,
                "speedup_vs_dense": (tokens_per_s / dense["value"]) if dense else None,
                "cpu_baseline": cpu,
                "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "tokens/s",
                        "h2d_bytes_per_step": int(qh.numel() * 4),
                        "d2h_bytes_per_step": int(oh.numel() * 4)},
                "gpu_launches": args.steps * (n_launch if fused else 2 * n_launch if world == 1
                                              else 2 * n_launch + 1),
                "clocks": clk, "prefill": W["timings"], "budget": W["info"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
