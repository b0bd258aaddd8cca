"""N > 1 host logic on CPU: the page-range split of one sequence across ranks
 and the two-level LSE merge, over a real world_size-2 gloo
process group.

Each rank takes `plan.split_ranges` of every (layer, kv-head) pointer list,
computes its split's softmax state with the oracle (decode.py:291-355 restated
on a page subset), converts it to the state form `sphkv_lse_merge_ex
(state_out=1)` emits (m = log-sum-exp, l = 1, acc = normalized output), and
all-gathers it rank-major exactly as bench.py does; the merge over ranks must
equal the single-pass reference softmax.  The device kernels for the same two
merge levels are parity-tested in tests/test_gpu_parity.py.
"""

import math
import os
import socket

import numpy as np
import pytest

from oracle import sphkv_oracle as O
from paper_2605_18856_b200.plan import split_ranges

TIERS = [(0, 0, 0, 0), (1, 2, 4, 8), (2, 4, 6, 8), (3, 12, 14, 8)]


def _store(seed=0, L=1, H=2, T=700, d=16, P=64):
    rng = np.random.default_rng(seed)
    keys = rng.standard_normal((L, H, T, d))
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    r, ang = O.encode_batch(keys.reshape(-1, d))
    tier = rng.choice([0, 1, 2, 3], (L, H, T), p=[0.1, 0.4, 0.3, 0.2]).astype(np.int16)
    z = (tier != 0).astype(np.int8)
    st = O.pack_pages(TIERS, z, tier, np.zeros((L, H, T), bool), r.reshape(L, H, T),
                      ang.reshape(L, H, T, d - 1), vals, P)
    q = rng.standard_normal((L, H, d)) * 4
    return st, q


def _page_stream_bytes(st, idx):
    ang, rad, val, _, _, _ = st.page_bytes(st.pages[idx])
    return 16 + ang + rad + val


def _range_state(st, l, h, q, begin, end):
    """Softmax state of pointer positions [begin, end) in the state_out form."""
    rq, qf = O.query_features(q[None])
    cache = O.FeatureCache()
    sub = O.OracleStore(st.tiers, st.layers, st.heads, st.d, st.d_v, st.page_size)
    sub.pages = st.pages
    sub.pointer = {k: [] for k in st.pointer}
    sub.pointer[(l, h)] = st.pointer[(l, h)][begin:end]
    logits, out = O.head_attend(sub, l, h, rq[0], qf[0], cache)
    if logits.size == 0:
        return -math.inf, 0.0, np.zeros(st.d_v)
    mx = logits.max()
    return mx + math.log(np.exp(logits - mx).sum()), 1.0, out


def _merge_rank_major(gathered, world, n_groups):
    """restates k_lse_merge with slot_begin == NULL: slot = g + s * n_groups."""
    out = []
    for g in range(n_groups):
        slots = [gathered[g + s * n_groups] for s in range(world)]
        m = np.array([x[0] for x in slots])
        lsum = np.array([x[1] for x in slots])
        acc = np.array([x[2] for x in slots])
        out.append(O.lse_merge(m, lsum, acc))
    return np.array(out)


def test_split_ranges_cover_and_balance():
    rng = np.random.default_rng(1)
    for n in (0, 1, 2, 7, 33, 200):
        b = rng.integers(1, 1000, n)
        for world in (1, 2, 3, 4, 8):
            rs = split_ranges(b, world)
            assert len(rs) == world
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (s0, e0), (s1, e1) in zip(rs[:-1], rs[1:]):
                assert e0 == s1 and s0 <= e0
            if n >= 4 * world:
                share = [int(b[s:e].sum()) for s, e in rs]
                assert max(share) <= b.sum() / world + b.max()


def test_split_merge_equals_single_pass_host():
    st, q = _store()
    for world in (1, 2, 3, 5):
        for (l, h) in st.pointer:
            lst = st.pointer[(l, h)]
            rs = split_ranges([_page_stream_bytes(st, i) for i in lst], world)
            states = [_range_state(st, l, h, q[l, h], s, e) for s, e in rs]
            got = _merge_rank_major(states, world, 1)[0]
            rq, qf = O.query_features(q[l, h][None])
            _, want = O.head_attend(st, l, h, rq[0], qf[0])
            assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    st, q = _store(seed=3)
    groups = sorted(st.pointer)
    F = 2 + st.d_v
    mine = np.zeros((len(groups), F))
    for gi, (l, h) in enumerate(groups):
        lst = st.pointer[(l, h)]
        s, e = split_ranges([_page_stream_bytes(st, i) for i in lst], world)[rank]
        m, lsum, acc = _range_state(st, l, h, q[l, h], s, e)
        mine[gi, 0], mine[gi, 1], mine[gi, 2:] = m, lsum, acc
    t = torch.from_numpy(mine.reshape(-1))
    gathered = torch.empty(world * t.numel(), dtype=t.dtype)
    dist.all_gather_into_tensor(gathered, t)
    g = gathered.numpy().reshape(world * len(groups), F)
    out = _merge_rank_major([(r[0], r[1], r[2:]) for r in g], world, len(groups))
    if rank == 0:
        np.save(result_path, out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_page_range_split(tmp_path):
    import torch.multiprocessing as mp

    world = 2
    res = str(tmp_path / "out.npy")
    mp.spawn(_worker, args=(world, _free_port(), res), nprocs=world, join=True)
    got = np.load(res)
    st, q = _store(seed=3)
    for gi, (l, h) in enumerate(sorted(st.pointer)):
        rq, qf = O.query_features(q[l, h][None])
        _, want = O.head_attend(st, l, h, rq[0], qf[0])
        assert np.max(np.abs(got[gi] - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


# ---------------------------------------------------------------------------
# batch x KV-head shards: ownership and per-sequence RDR
# ---------------------------------------------------------------------------

def test_shard_ownership_covers_every_pair_once():
    import bench

    for B, H in ((16, 8), (8, 8), (4, 8), (1, 8), (3, 5)):
        for world in (1, 2, 3, 4, 8):
            owned = [bench.owned_pairs(B, H, r, world, "shard") for r in range(world)]
            flat = [p for o in owned for p in o]
            assert sorted(flat) == [(b, h) for b in range(B) for h in range(H)]
            for o in owned:  # a rank's heads of one sequence are a contiguous range
                for b in {p[0] for p in o}:
                    hs = sorted(h for bb, h in o if bb == b)
                    assert hs == list(range(hs[0], hs[-1] + 1))


def _alloc_worker(rank, world, port, result_path):
    """Each rank holding part of sequence 0 runs the SAME per-sequence RDR
    allocation (oracle score + greedy, controller.py:213-346) on the whole
    sequence and keeps its own heads; the gathered decisions must agree."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)  # the sequence's data: identical on every rank
    L, H, T, d = 2, 4, 300, 16
    radii = np.abs(rng.standard_normal((L, H, T))) + 0.5
    eps = {1: (0.08, 0.02), 2: (0.02, 0.005), 3: (0.001, 0.0003)}
    seg = np.full(T, 2, np.int8)
    seg[:200] = 0
    prot = np.zeros((L, H, T), bool)
    sc = O.score_states(radii, rng.uniform(0.2, 1, (L, H)), rng.uniform(0, 0.8, (L, H)), 30.0,
                        (0.02, 2.0, 1.0), seg, 1.0, 1.0, TIERS, eps, 3e-5, prot, d)
    z, tier = O.allocate_greedy(sc["best_tier"], sc["nu"], prot, int(0.3 * L * H * T * d * 16),
                                TIERS, d)
    t = torch.from_numpy(tier.astype(np.int64).reshape(-1))
    g = torch.empty(world * t.numel(), dtype=t.dtype)
    dist.all_gather_into_tensor(g, t)
    if rank == 0:
        np.save(result_path, g.numpy().reshape(world, -1))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_replicated_sequence_allocation(tmp_path):
    import torch.multiprocessing as mp

    res = str(tmp_path / "alloc.npy")
    mp.spawn(_alloc_worker, args=(2, _free_port(), res), nprocs=2, join=True)
    got = np.load(res)
    assert np.array_equal(got[0], got[1]) and np.any(got[0] == 0) and np.any(got[0] > 0)


def _device_worker(rank, world, port, result_path):
    """Both ranks on cuda:0 over gloo: device page-range decode of the rank's
    share (fused state output), all-gather of the states, device merge."""
    import torch
    import torch.distributed as dist
    import paper_2605_18856_b200 as sk
    from paper_2605_18856_b200 import plan as planmod

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    st, q, tl = _device_store(sk)
    groups = list(range(st.groups))
    p = planmod.plan_store_range(st, groups, rank, world, grid=16)
    state = sk.decode.ada_decode_state(st, q, p).cpu()
    gathered = torch.empty((world,) + tuple(state.shape), dtype=state.dtype)
    dist.all_gather_into_tensor(gathered.view(-1), state.view(-1))
    G, dv = q.shape[1], st.d_v
    out = torch.empty((len(groups) * G, dv), dtype=torch.float32, device="cuda")
    planmod.merge_gathered(len(groups), world, gathered.cuda(), G, dv, out)
    if rank == 0:
        np.save(result_path, out.double().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _device_store(sk):
    import torch

    rng = np.random.default_rng(5)
    L, H, T, d, G, P = 2, 2, 2500, 64, 4, 128
    keys = rng.standard_normal((L, H, T, d))
    vals = rng.standard_normal((L, H, T, d)).astype(np.float16).astype(np.float64)
    r, ang = O.encode_batch(keys.reshape(-1, d))
    tier = rng.choice([0, 1, 2, 3], (L, H, T), p=[0.1, 0.4, 0.3, 0.2]).astype(np.int16)
    tiers = sk.TierTable(tuple(sk.TierSpec(*t) for t in TIERS))
    st = sk.pack_pages_arrays(sk.TierAssignment((tier != 0).astype(np.int8), tier,
                                                np.zeros((L, H, T), bool)),
                              r.reshape(L, H, T), ang.reshape(L, H, T, d - 1), vals, tiers, P)
    q = torch.as_tensor(rng.standard_normal((L * H, G, d)) * 4, dtype=torch.float32,
                        device="cuda")
    return st, q, TIERS


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_gloo_world2_device_page_range_split(tmp_path):
    """The N > 1 page-range data path through the DEVICE kernels: two gloo
    ranks (both on the one GPU) decode their shares, all-gather the states and
    merge; equals the single-pass device decode and the oracle."""
    import torch
    import torch.multiprocessing as mp
    import paper_2605_18856_b200 as sk

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    res = str(tmp_path / "dev.npy")
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_device_worker, args=(r, 2, _free_port_shared(), res))
             for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=500)
        assert pr.exitcode == 0
    got = np.load(res)
    st, q, _ = _device_store(sk)
    want = sk.ada_decode(st, q, sk.plan_store(st)).double().cpu().numpy()
    assert np.max(np.abs(got - want)) <= 2e-5 * max(1.0, np.abs(want).max())


_PORT = None


def _free_port_shared():
    global _PORT
    if _PORT is None:
        _PORT = _free_port()
    return _PORT
