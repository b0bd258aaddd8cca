"""A1 ablation (PAPER reconstruct-then-dot, decode.py:195-217) on one c5 layer:
time the dense staging write (sphkv_recon_keys, fp16 rows) plus the dot's
re-read (cuBLAS GEMV over the staged rows, all G query heads) against the ADA
kernel on the same pages.  The staged bytes are the densification tax."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
import paper_2605_18856_b200 as sk
from paper_2605_18856_b200 import _lib, plan as planmod

W = bench.build_workload("c5", dense=False, parity=False)
st, qall = W["st"], W["q"]
B, L, H, G, T, d, _ = bench.CONFIGS["c5"]
groups = [(b * L + 0) * H + h for b in range(B) for h in range(H)]
n, rows, plen, ptr = st._host()
pids = np.concatenate([ptr[g, : plen[g]] for g in groups]).astype(np.int32)
counts = rows["count"][pids].astype(np.int64)
off = np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)
items = int(counts.sum())
stage = torch.empty((items, d), dtype=torch.float16, device="cuda")
pid_t, off_t = torch.as_tensor(pids, device="cuda"), torch.as_tensor(off, device="cuda")
lib = _lib.lib()
per_group = [int(rows["count"][ptr[g, : plen[g]]].sum()) for g in groups]
bounds = np.concatenate([[0], np.cumsum(per_group)]).astype(np.int64)
dot_out = torch.empty((items, G), dtype=torch.float32, device="cuda")


def recon():  # staging write: every item's key decoded to fp16 rows (sphkv_recon_keys)
    _lib.check(lib.sphkv_recon_keys(st.cptr, pid_t.data_ptr(), off_t.data_ptr(), len(pids),
                                    stage.data_ptr(), _lib.F16, _lib.stream_ptr()))


def reread():  # the dot's re-read of the staged rows, G query heads (sphkv_recon_dot)
    for k, g in enumerate(groups):
        a, b = int(bounds[k]), int(bounds[k + 1])
        _lib.check(lib.sphkv_recon_dot(stage[a:b].data_ptr(), _lib.F16, b - a, d, qall[g].data_ptr(),
                                       G, dot_out[a:b].data_ptr(), _lib.stream_ptr()))


def timeit(fn, it=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3


p = planmod.plan_store(st, groups=groups, units_per_cta=1)
out = torch.empty((len(groups) * G, d), dtype=torch.float32, device="cuda")
t_ada = timeit(lambda: sk.ada_decode(st, qall, p, out=out))
t_w = timeit(recon)
t_r = timeit(reread)
tax = items * d * 2
print(f"items {items}: ADA decode {t_ada:.1f} us; recon staging write {t_w:.1f} us "
      f"({tax / t_w / 1e3:.0f} GB/s of staged rows); re-read dot {t_r:.1f} us; "
      f"densification tax {tax / 1e6:.1f} MB each way = {2 * tax / st.stream_bytes_total() * L:.2f}x "
      f"the layer's ADA stream bytes")
