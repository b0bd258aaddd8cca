"""LSB-first fixed-width code streams (drop-in for sphkv.bitpack, bitpack.py:14-48).

The device writes these streams directly into pages (encode_pack.cu); this
host module is the file-format utility used for SPHKV1 snapshots and for
inspecting exported pages.
"""

from __future__ import annotations

import numpy as np


def packed_nbytes(count: int, bits: int) -> int:
    return (count * bits + 7) // 8


def pack_bits(codes, bits: int) -> np.ndarray:
    codes = np.asarray(codes, dtype=np.uint64).ravel()
    if bits < 1 or bits > 64:
        raise ValueError(f"bits must be in [1, 64], got {bits}")
    if codes.size and bits < 64 and int(codes.max()) >> bits:
        raise ValueError(f"code does not fit in {bits} bits")
    if codes.size == 0:
        return np.zeros(0, dtype=np.uint8)
    planes = ((codes[:, None] >> np.arange(bits, dtype=np.uint64)[None, :])
              & np.uint64(1)).astype(np.uint8)
    return np.packbits(planes.ravel(), bitorder="little")[: packed_nbytes(codes.size, bits)]


def unpack_bits(stream, bits: int, count: int) -> np.ndarray:
    stream = np.asarray(stream, dtype=np.uint8)
    if packed_nbytes(count, bits) > stream.size:
        raise ValueError("stream too short for requested codes")
    flat = np.unpackbits(stream, bitorder="little")[: count * bits]
    planes = flat.reshape(count, bits).astype(np.uint64)
    return (planes << np.arange(bits, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
