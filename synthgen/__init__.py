"""Seeded, counter-based synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic (no ordering, aggregation,
commit or replication math).  It only turns (seed, stream, counter) into numbers:

* update vectors and the initial model w0 (the values the GPU path and the
  oracle both consume), and
* the harness's scenario draws: NIC rates from the paper's N1-N3 presets
  (§7 "Background compute and network load"), C1-C3
  straggler draws, and the seeded random aggregator
  pre-assignment the paper leaves to the caller (§5.2
  "We first randomly pre-assign the aggregator"; reading R13 in DESIGN.md).

The counter-based generator is splitmix64 (Steele, Lea, Flood 2014):
    word(key, i) = mix64(key + (i + 1) * 0x9E3779B97F4A7C15  mod 2^64)
The CUDA library implements the same function independently in
``paper_1907_00434_b200/csrc/synth.cu`` (``mlf_synth_fill``); the two share no
code, and ``tests/test_synthgen.py`` / the GPU tests check they agree bit for bit.

Value maps (all exactly representable, so no rounding ever happens while
generating):
  variant "normal":  fp32 update = int24 * 2^-31    (int24 = (word >> 40) - 2^23)
                     bf16 update = int8  * 2^-14    (int8  = (word >> 56) - 128)
                     w0          = int24 * 2^-24
  variant "exact":   fp32 update = int11 * 2^-20    (int11 = (word >> 53) - 1024)
                     bf16 update = int8  * 2^-17
                     w0          = int22 * 2^-24    (int22 = (word >> 42) - 2^21)
The "exact" variant is the exact-arithmetic special case of SURVEY.md §8(c) O6:
every sum / product / difference the commit performs is exact in fp32 for
<= 256 updates per batch and <= 20 batches, so any summation order gives the
same bits.
"""
from __future__ import annotations

import numpy as np

SEED_ROOT = 0x4D4C46  # "MLF"
GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1

# stream kinds (first key component)
KIND_UPDATE = 1
KIND_W0 = 2
KIND_NET = 3
KIND_STRAGGLER = 4
KIND_AGG_SHUFFLE = 5
KIND_MISC = 6

VARIANT_NORMAL = 0
VARIANT_EXACT = 1
_VARIANTS = {"normal": VARIANT_NORMAL, "exact": VARIANT_EXACT}

DTYPE_F32 = 0
DTYPE_BF16 = 1


# ----------------------------------------------------------------- scalar core
def mix64(z: int) -> int:
    """splitmix64 finaliser on a Python int (mod 2^64)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def sm64(x: int) -> int:
    """One splitmix64 step from state x: mix64(x + GOLDEN)."""
    return mix64((x + GOLDEN) & MASK64)


def stream_key(seed: int, kind: int, a: int = 0, b: int = 0) -> int:
    """Key of the stream (seed, kind, a, b)."""
    k = sm64((seed & MASK64) ^ (kind & MASK64))
    k = sm64(k ^ (a & MASK64))
    return sm64(k ^ (b & MASK64))


def word(key: int, i: int) -> int:
    """The i-th 64-bit word of stream `key`."""
    return mix64((key + (i + 1) * GOLDEN) & MASK64)


# ------------------------------------------------------------- vectorised core
def words(key: int, idx) -> np.ndarray:
    """word(key, i) for every i in idx (uint64 array), vectorised."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (idx + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def _ints(w: np.ndarray, shift: int, bias: int) -> np.ndarray:
    return (w >> np.uint64(shift)).astype(np.int64) - bias


def _f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    # exact for the values generated here (<= 8 significant bits)
    b = x.astype(np.float32).view(np.uint32)
    assert not np.any(b & np.uint32(0xFFFF)), "value not exactly representable in bf16"
    return (b >> np.uint32(16)).astype(np.uint16)


def update_values(seed: int, worker: int, iteration: int, idx, dtype: int = DTYPE_F32,
                  variant: str = "normal") -> np.ndarray:
    """Elements `idx` of worker `worker`'s update in iteration `iteration`.

    Returns float32 values (dtype F32) or uint16 bf16 bit patterns (dtype BF16).
    """
    v = _VARIANTS[variant]
    w = words(stream_key(seed, KIND_UPDATE, worker, iteration), idx)
    if dtype == DTYPE_F32:
        if v == VARIANT_NORMAL:
            return np.ldexp(_ints(w, 40, 1 << 23).astype(np.float64), -31).astype(np.float32)
        return np.ldexp(_ints(w, 53, 1024).astype(np.float64), -20).astype(np.float32)
    if dtype == DTYPE_BF16:
        scale = -14 if v == VARIANT_NORMAL else -17
        return _f32_to_bf16_bits(np.ldexp(_ints(w, 56, 128).astype(np.float64), scale))
    raise ValueError(dtype)


def w0_values(seed: int, idx, variant: str = "normal") -> np.ndarray:
    """Elements `idx` of the initial model w0 (float32)."""
    v = _VARIANTS[variant]
    w = words(stream_key(seed, KIND_W0, 0, 0), idx)
    if v == VARIANT_NORMAL:
        return np.ldexp(_ints(w, 40, 1 << 23).astype(np.float64), -24).astype(np.float32)
    return np.ldexp(_ints(w, 42, 1 << 21).astype(np.float64), -24).astype(np.float32)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Widen bf16 bit patterns to float32 (u32 = u16 << 16), exact."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ------------------------------------------------------------- scenario draws
GBPS = 1_000_000_000 // 8  # bytes/s per Gb/s
RATE_SET_BPS = (125_000_000, 312_500_000, 412_500_000, 625_000_000, 1_250_000_000)
# rate set {1, 2.5, 3.3, 5, 10} Gb/s with probabilities p
N_PRESETS = {
    "N1": (0.0, 0.0, 0.0, 0.1, 0.9),
    "N2": (0.0, 0.1, 0.1, 0.1, 0.7),
    "N3": (0.5, 0.0, 0.0, 0.0, 0.5),
}
# (r %, s)
C_PRESETS = {"C1": (10, 2), "C2": (10, 4), "C3": (4, 2)}


def uniform01(key: int, i: int) -> float:
    """A double in [0, 1) from the top 53 bits of word(key, i)."""
    return (word(key, i) >> 11) * (1.0 / (1 << 53))


def draw_rate(key: int, i: int, preset: str) -> int:
    """One NIC rate (bytes/s) drawn from an N-preset's probability vector."""
    u = uniform01(key, i)
    acc = 0.0
    probs = N_PRESETS[preset]
    for r, p in zip(RATE_SET_BPS, probs):
        acc += p
        if u < acc:
            return r
    # u lands beyond the rounded cumulative sum: the last non-zero entry
    for r, p in reversed(list(zip(RATE_SET_BPS, probs))):
        if p > 0:
            return r
    raise ValueError(preset)


def draw_rates(seed: int, n: int, preset: str, epoch: int = 0, salt: int = 0) -> list[int]:
    key = stream_key(seed, KIND_NET, epoch, salt)
    return [draw_rate(key, i, preset) for i in range(n)]


def draw_stragglers(seed: int, n: int, preset: str, iteration: int) -> list[int]:
    """Per-worker slowdown factor (1 or s) for one iteration, C-preset (r %, s)."""
    r, s = C_PRESETS[preset]
    key = stream_key(seed, KIND_STRAGGLER, iteration, 0)
    return [s if uniform01(key, i) * 100.0 < r else 1 for i in range(n)]


def shuffle(seed: int, items, salt: int = 0) -> list:
    """Seeded Fisher-Yates shuffle (splitmix64 words; j = word mod (i+1))."""
    out = list(items)
    key = stream_key(seed, KIND_AGG_SHUFFLE, salt, 0)
    for i in range(len(out) - 1, 0, -1):
        j = word(key, i) % (i + 1)
        out[i], out[j] = out[j], out[i]
    return out


def randint(key: int, i: int, lo: int, hi: int) -> int:
    """Integer in [lo, hi] (inclusive) from word(key, i) (modulo draw)."""
    return lo + word(key, i) % (hi - lo + 1)
