"""ORACLE / TEST INFRASTRUCTURE ONLY -- the deterministic counter-hash payloads.

Mirrors oracle/ref_tool.cpp (piece_value) and the product's CUDA fill kernel
(paper_2504_20490_b200/csrc/exec/datagen.cuh).  Every stored value is a pure
function of (seed, tensor id, piece, global linear index), so any box of any
shard can be regenerated independently on CPU or GPU (SURVEY §8d "Synthetic
inputs").

mode "grid": exact small integers.  The logical tensor X is gv(h) in [-4, 4);
  a top-tier Partial (effective hdim -2) splits X into hsize pieces and a
  bottom Partial of count P splits each piece into P pieces; the last piece is
  the remainder, so every decomposition sums EXACTLY to X in any dtype (all
  partial sums stay far inside bf16's exact-integer range).
mode "real": uniform [-1, 1) with 23 fractional bits, pieces independent (sums
  exercise rounding; only bit-exact comparisons with the same reduction order
  are meaningful).
"""
from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)


def _u32(x):
    return np.asarray(x, dtype=np.uint64) & M32


def mix32(x):
    x = _u32(x)
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & M32
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & M32
    x ^= x >> np.uint64(16)
    return x


def hash3(seed: int, key: int, lin):
    """ref_tool.cpp hash3: three rounds of mix32 over (seed, key, lin lo, lin hi)."""
    lin = np.asarray(lin, dtype=np.uint64)
    h0 = (int(seed) * 0x9E3779B1 + int(key) * 0x85EBCA77 + 0x165667B1) & 0xFFFFFFFF
    h = mix32(np.uint64(h0))
    h = mix32(h ^ (lin & M32))
    h = mix32(h ^ (lin >> np.uint64(32)) ^ np.uint64(0x27D4EB2F))
    return h


def piece_key(tensor_id: int, level: int, g: int, p: int) -> int:
    return (tensor_id * 1000003 + level * 7919 + g * 131 + p) & 0xFFFFFFFF


def grid_value(h):
    return ((h >> np.uint64(8)) % np.uint64(8)).astype(np.int64) - 4


def real_value(h):
    return ((h >> np.uint64(8)).astype(np.float64) * 2.0 ** -23 - 1.0).astype(np.float32)


def f32_to_bf16_bits(x):
    """Round-to-nearest-even float32 -> bfloat16 bit pattern (uint16)."""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


NP_DTYPE = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64,
            "bf16": np.uint16}


def encode(values, dtype: str):
    """float64 / int64 values -> storage array of `dtype` (bf16 as raw uint16)."""
    if dtype == "bf16":
        return f32_to_bf16_bits(np.asarray(values, dtype=np.float32))
    return np.asarray(values).astype(NP_DTYPE[dtype])


def decode(arr, dtype: str):
    """storage -> float64 (exact for the grid)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(arr).astype(np.float64)
    return np.asarray(arr).astype(np.float64)


def logical_grid(lin, seed: int, tid: int):
    return grid_value(hash3(seed, piece_key(tid, 0, 0, 0), lin))


def piece_grid(lin, seed, tid, hsize, tg, g, p, P):
    """Exact integer stored by a device (ref_tool.cpp piece_value)."""
    x = logical_grid(lin, seed, tid)
    if tg >= 0:
        if tg < hsize - 1:
            t = grid_value(hash3(seed, piece_key(tid, 1, tg, 0), lin))
        else:
            s = np.zeros_like(x)
            for k in range(hsize - 1):
                s = s + grid_value(hash3(seed, piece_key(tid, 1, k, 0), lin))
            t = x - s
    else:
        t = x
    if P == 1:
        return t
    if p < P - 1:
        return grid_value(hash3(seed, piece_key(tid, 2, g, p), lin))
    s = np.zeros_like(x)
    for k in range(P - 1):
        s = s + grid_value(hash3(seed, piece_key(tid, 2, g, k), lin))
    return t - s


def piece_real(lin, seed, tid, tg, p):
    return real_value(hash3(seed, piece_key(tid, 3, tg + 1, p), lin))


def box_linear_indices(shape, bounds):
    """Global row-major linear index of every cell of `bounds`, in box row-major order."""
    shape = [int(s) for s in shape]
    strides = np.ones(len(shape), dtype=np.int64)
    for i in range(len(shape) - 2, -1, -1):
        strides[i] = strides[i + 1] * shape[i + 1]
    lin = np.zeros([hi - lo for lo, hi in bounds], dtype=np.int64)
    for d, (lo, hi) in enumerate(bounds):
        idx = np.arange(lo, hi, dtype=np.int64) * strides[d]
        sh = [1] * len(bounds)
        sh[d] = hi - lo
        lin = lin + idx.reshape(sh)
    return lin.astype(np.uint64)


def shard_values(shape, bounds, seed, tid, hsize, tg, g, p, P, dtype, mode="grid"):
    lin = box_linear_indices(shape, bounds)
    if mode == "grid" or dtype in ("i32", "i64"):
        return encode(piece_grid(lin, seed, tid, hsize, tg, g, p, P), dtype)
    return encode(piece_real(lin, seed, tid, tg, p), dtype)
