"""ctypes binding of libsphkv_b200.so (the C ABI in include/sphkv_b200.h).

There is no CPU fallback: `lib()` raises if the shared library is missing or
no sm_100 device is visible, and every wrapper raises on a non-zero status
with the reference's exception types.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_double, c_int, c_int32, c_int64, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPHKV_LIB") or os.path.join(HERE, "libsphkv_b200.so")

SPHKV_OK = 0
SPHKV_E_VALUE = 1
SPHKV_E_KEY = 2
SPHKV_E_INFEASIBLE = 3
SPHKV_E_UNSUPPORTED = 4
SPHKV_E_CUDA = 5
SPHKV_E_CAPACITY = 6

F32, F64, BF16, F16 = 0, 1, 2, 3
LIVE_AFTER_MUTATION, LIVE_ABS_ROWS = 1, 2
MAX_TIERS = 16


class InfeasibleProtectionError(Exception):
    """Protected demand alone exceeds the bit budget (controller.py:46-47)."""


class CTier(ctypes.Structure):
    _fields_ = [("id", c_int32), ("angle_bits", c_int32), ("radius_bits", c_int32),
                ("meta_bits", c_int32), ("eps_theta", c_double), ("eps_r", c_double)]


class CStore(ctypes.Structure):
    _fields_ = [("batch", c_int32), ("layers", c_int32), ("heads", c_int32), ("d", c_int32),
                ("d_v", c_int32), ("page_size", c_int32), ("n_tiers", c_int32),
                ("max_pages", c_int32), ("ptr_cap", c_int32), ("lut_flags", c_int32),
                ("code_cap", c_uint64), ("tiers", CTier * MAX_TIERS),
                ("pages", c_void_p), ("ptr", c_void_p), ("ptr_len", c_void_p),
                ("group_last", c_void_p), ("codes", c_void_p), ("values", c_void_p),
                ("protect", c_void_p), ("token_ids", c_void_p), ("counters", c_void_p),
                ("lut", c_void_p), ("lut_off", c_int32 * MAX_TIERS),
                ("lut_items", ctypes.c_int64 * MAX_TIERS)]


class CDenseStore(ctypes.Structure):
    _fields_ = [("batch", c_int32), ("layers", c_int32), ("heads", c_int32), ("d", c_int32),
                ("d_v", c_int32), ("page_size", c_int32), ("n_pages_per_group", c_int32),
                ("tokens", c_int32), ("keys", c_void_p), ("values", c_void_p)]


# device page descriptor, 32 bytes (sphkv_page_t)
PAGE_DTYPE = np.dtype([("code_off", "<u8"), ("radius_scale", "<f8"), ("rscale", "<f4"),
                       ("count", "<i4"), ("group", "<i4"), ("tier", "u1"), ("abits", "u1"),
                       ("rbits", "u1"), ("mbits", "u1")])
assert PAGE_DTYPE.itemsize == 32
UNIT_DTYPE = np.dtype([("group", "<i4"), ("ptr_begin", "<i4"), ("ptr_end", "<i4"),
                       ("out_slot", "<i4")])

_LIB = None


def _declare(lib):
    vp, i, i64, d = c_void_p, c_int, c_int64, c_double
    sig = {
        "sphkv_abi_version": (c_int, []),
        "sphkv_last_error": (ctypes.c_char_p, []),
        "sphkv_device_ok": (c_int, []),
        "sphkv_encode_radii": (c_int, [vp, i, i64, i, vp, vp]),
        "sphkv_encode": (c_int, [vp, i, i64, i, vp, vp, vp]),
        "sphkv_quantize_angles": (c_int, [vp, i64, i, i, vp, vp]),
        "sphkv_angles_from_unit": (c_int, [vp, i64, i, vp, vp]),
        "sphkv_rdr_score": (c_int, [vp, vp, vp, vp, d, d, d, vp, i, d, vp, i, i, i, i,
                                    vp, vp, vp, vp, vp]),
        "sphkv_rdr_workspace_bytes": (c_int64, [i64]),
        "sphkv_rdr_allocate_greedy": (c_int, [vp, vp, vp, i64, vp, i, i, i64, vp, vp, vp, vp]),
        "sphkv_rdr_downtier": (c_int, [vp, vp, vp, i64, vp, i, i, i64, vp, vp, vp, vp]),
        "sphkv_store_reset": (c_int, [vp, vp]),
        "sphkv_lut_floats": (c_int64, [vp]),
        "sphkv_ada_tile_items": (c_int, []),
        "sphkv_unit_tile_cap": (c_int, []),
        "sphkv_store_build_lut": (c_int, [vp, vp]),
        "sphkv_pack_pages": (c_int, [vp, vp, i, vp, vp, vp, vp, vp, vp, i, vp, i64, vp]),
        "sphkv_pack_workspace_bytes": (c_int64, [i, i, i, i]),
        "sphkv_pack_pages_groups": (c_int, [vp, i, i, vp, i, vp, vp, vp, vp, vp, vp, i, vp, i64,
                                            vp]),
        "sphkv_append": (c_int, [vp, vp, i, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "sphkv_append_workspace_bytes": (c_int64, [i]),
        "sphkv_score_append": (c_int, [vp, i, i, vp, vp, d, d, d, d, vp, i, d, i, i64,
                                       vp, vp, vp, vp]),
        "sphkv_export_streams": (c_int, [vp, i, vp, vp, vp]),
        "sphkv_import_streams": (c_int, [vp, i, vp, vp, vp]),
        "sphkv_dense_fill": (c_int, [vp, vp, i, vp, vp]),
        "sphkv_dense_fill_groups": (c_int, [vp, i, i, vp, i, vp, vp]),
        "sphkv_ada_decode": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp]),
        "sphkv_dense_decode": (c_int, [vp, vp, i, vp, i, vp, i, vp]),
        "sphkv_lse_merge": (c_int, [vp, vp, i, i, i, vp, vp]),
        "sphkv_lse_merge_ex": (c_int, [vp, vp, i, i64, i, i, i, vp, i, vp]),
        "sphkv_recon_keys": (c_int, [vp, vp, vp, i, vp, i, vp]),
        "sphkv_ada_decode_margins": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, i, vp, vp,
                                             i, vp]),
        "sphkv_ada_decode_fused": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, i, i, vp]),
        "sphkv_ada_decode_state": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, i, vp]),
        "sphkv_ada_decode_live": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, vp, vp, i, i,
                                          vp]),
        "sphkv_dense_decode_fused": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, i, i, vp]),
        "sphkv_dense_decode_window": (c_int, [vp, vp, i, vp, i, vp, vp, vp, i, vp, vp, i, i, i,
                                              vp]),
        "sphkv_partial_floats": (c_int64, [i, i]),
        "sphkv_f64_to_f16": (c_int, [vp, i64, vp, vp]),
        "sphkv_controller_workspace_bytes": (c_int64, [i64, i]),
        "sphkv_controller_stats": (c_int, [vp, i, vp, vp, i, i64, i, i, i, i, vp, vp, vp, vp]),
        "sphkv_decode_gate": (c_int, [vp, vp, i, vp, i, vp, vp, vp, d, d, d, d, d, i, d, d, d,
                                      vp, vp, vp, vp, vp]),
        "sphkv_recon_dot": (c_int, [vp, i, i64, i, vp, i, vp, vp]),
        "sphkv_dense_logits": (c_int, [vp, vp, i64, i, vp, vp]),
        "sphkv_dense_store_logits": (c_int, [vp, vp, i, i, vp, vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("SPHKV_LIB") and not hasattr(lib, name):
            continue  # experiment builds (SPHKV_LIB) may predate newer entry points
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """Load the extension (built in-tree); raise loudly when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (no CPU fallback exists)")
    import torch  # noqa: F401  -- loads the CUDA runtime the library links against
    l = ctypes.CDLL(LIB_PATH)
    _declare(l)
    if l.sphkv_abi_version() != 1:
        raise RuntimeError("libsphkv_b200 ABI mismatch")
    _LIB = l
    return l


def require_gpu():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_18856_b200 needs a CUDA B200 (sm_100) device; "
                           "there is no CPU fallback")
    l = lib()
    if not l.sphkv_device_ok():
        raise RuntimeError("current CUDA device is not sm_100 (B200)")
    return l


def check(status: int):
    if status == SPHKV_OK:
        return
    msg = (_LIB.sphkv_last_error() or b"").decode(errors="replace")
    if status in (SPHKV_E_VALUE, SPHKV_E_UNSUPPORTED):
        raise ValueError(msg)
    if status == SPHKV_E_KEY:
        raise KeyError(msg)
    if status == SPHKV_E_INFEASIBLE:
        raise InfeasibleProtectionError(msg)
    raise RuntimeError(f"sphkv error {status}: {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def tiers_to_c(tiers) -> "CTier * MAX_TIERS":
    arr = (CTier * MAX_TIERS)()
    for k, t in enumerate(tiers.tiers):
        et, er = (1.0, 1.0)
        if t.id != 0:
            et = tiers.eps_theta.get(t.id, 0.0)
            er = tiers.eps_r.get(t.id, 0.0)
        arr[k] = CTier(t.id, t.angle_bits, t.radius_bits, t.meta_bits, et, er)
    return arr


def to_f16(x):
    """Values -> fp16 device tensor with ONE round-to-nearest-even from the
    source type (numpy astype(np.float16) semantics, store.py:383): numpy
    input is rounded on the host; a float64 device tensor goes through
    sphkv_f64_to_f16 (torch's double->half rounds through fp32)."""
    import torch

    if isinstance(x, torch.Tensor):
        x = x.to("cuda").contiguous()
        if x.dtype != torch.float64:
            return x.to(torch.float16)  # fp32/bf16/fp16: one rounding
        out = torch.empty(x.shape, dtype=torch.float16, device="cuda")
        check(require_gpu().sphkv_f64_to_f16(x.data_ptr(), x.numel(), out.data_ptr(),
                                             stream_ptr()))
        return out
    a = np.asarray(x)
    if a.dtype != np.float16:
        a = a.astype(np.float64).astype(np.float16)
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")
