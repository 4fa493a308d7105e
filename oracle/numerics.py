"""Bit-level numerics shared by the oracle and the CUDA kernels.

TEST INFRASTRUCTURE (see oracle/__init__.py): the CUDA kernels implement the
same formulas; this module is the checker.

* Half rounding is round-to-nearest-even ("round-to-nearest-even
  binary16 of fp32 master", "cast to fp16 with
  round-to-nearest-even"). bfloat16 is the build's second half type
  (SURVEY.md §7 "Hard parts: fp16 vs bf16").
* Parameter init is "seeded uniform(-1/sqrt(in_dim), +1/sqrt(in_dim))
  generated in fp32 then rounded to fp16 ... deterministic per layer index"
  (SPEC.md:785). The generator is a counter-based splitmix64 hash of
  (seed, stream, element index) so that every rank can materialise only its
  own shard ("never fully instantiated") and the GPU kernel
  reproduces the oracle bit-for-bit.
"""

from __future__ import annotations

import math

import numpy as np

HALF_FP16 = 0
HALF_BF16 = 1

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


def half_dtype_name(kind: int) -> str:
    return {HALF_FP16: "fp16", HALF_BF16: "bf16"}[kind]


# ---------------------------------------------------------------- half casts

def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bfloat16 bit pattern (uint16), round-to-nearest-even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    bias = ((u >> 16) & 1) + 0x7FFF
    r = ((u + bias) >> 16).astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        r[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_half_bits(x: np.ndarray, kind: int) -> np.ndarray:
    """fp32 -> half bit pattern (uint16) for kind in {HALF_FP16, HALF_BF16}."""
    if kind == HALF_FP16:
        return np.ascontiguousarray(x, dtype=np.float32).astype(np.float16).view(np.uint16)
    if kind == HALF_BF16:
        return f32_to_bf16_bits(x)
    raise ValueError(f"unknown half kind {kind}")


def half_bits_to_f32(b: np.ndarray, kind: int) -> np.ndarray:
    if kind == HALF_FP16:
        return np.ascontiguousarray(b, dtype=np.uint16).view(np.float16).astype(np.float32)
    if kind == HALF_BF16:
        return bf16_bits_to_f32(b)
    raise ValueError(f"unknown half kind {kind}")


def round_half(x: np.ndarray, kind: int) -> np.ndarray:
    """fp32 -> nearest half (RNE) -> back to fp32."""
    return half_bits_to_f32(f32_to_half_bits(x, kind), kind)


# ---------------------------------------------------------------- counter RNG

def _mix_int(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def rng_key(seed: int, stream: int) -> int:
    """64-bit key of one generator stream (one per parameter tensor)."""
    return _mix_int(((seed * _GOLDEN) & _MASK) ^ _mix_int(stream + 0x632BE59BD9B4E019))


def _mix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


def rng_bits24(key: int, start: int, count: int) -> np.ndarray:
    """24-bit integers for element indices [start, start+count) of a stream."""
    idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + idx * np.uint64(_GOLDEN)
    return (_mix_np(z) >> np.uint64(40)).astype(np.int64)


def uniform_scale(bound: float) -> np.float32:
    """fp32 multiplier s such that x = float32(2k+1-2^24) * s lies in (-bound, bound)."""
    return np.float32(bound * 2.0 ** -24)


def init_bound(fan_in: int) -> float:
    return 1.0 / math.sqrt(fan_in)


def uniform_init(seed: int, stream: int, start: int, count: int, bound: float) -> np.ndarray:
    """fp32 U(-bound, bound) values for elements [start, start+count) of a stream.

    Mirrors kernel ``zi_init_uniform`` (paper_2104_07857_b200/csrc/init.cu):
    v = 2k + 1 - 2^24 is an odd integer exactly representable in fp32, and the
    single fp32 multiply by s rounds identically on both sides.
    """
    k = rng_bits24(rng_key(seed, stream), start, count)
    v = (2 * k + 1 - (1 << 24)).astype(np.float32)
    return v * uniform_scale(bound)
