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
