"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no projection, attention or
all-to-all). It only maps (seed, tensor_id, global element index) to a value,
so that both sides can draw the same inputs:

* the oracle and the tests call :func:`draw` (numpy, host);
* the CUDA path has its own implementation of the same counter-based generator
  (``paper_2602_21196_b200/csrc/misc.cu:synth_kernel``, exported as ``upipe_synth_fill_bf16``),
  used by ``bench.py`` to create large inputs directly in HBM.

Generator:

    z  = seed * 0x9E3779B97F4A7C15 + tensor_id * 0xD1B54A32D192ED03 + index   (mod 2^64)
    z  = splitmix64_finalize(z)
    m  = z >> 56                          (0 .. 255)
    v  = (2*m - 255) / 256 * 2**exponent

``v`` has at most 8 significant bits, so it is exactly representable in bf16,
fp32 and fp64: host and device values are bitwise identical with no rounding
step at all. The distribution is uniform on 256 odd levels in (-2^e, 2^e), i.e.
standard deviation ~ 2^e / sqrt(3).

Tensor ids (global indexing so sequence sharding cannot change values):
    X=1, Wq=2, Wk=3, Wv=4, Wo=5, dY=6 ; attention-core tests: Q=11, K=12, V=13, dO=14.
"""
from __future__ import annotations

import math

import numpy as np

TID = {"x": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "dy": 6,
       "q": 11, "k": 12, "v": 13, "do": 14, "q_norm_w": 7, "k_norm_w": 8}

_M64 = (1 << 64) - 1
_G1 = 0x9E3779B97F4A7C15
_G2 = 0xD1B54A32D192ED03


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(0xBF58476D1CE4E5B9)
    z ^= z >> np.uint64(27)
    z *= np.uint64(0x94D049BB133111EB)
    z ^= z >> np.uint64(31)
    return z


def draw_codes(seed: int, tensor_id: int, start: int, count: int) -> np.ndarray:
    """Raw 8-bit codes m in [0, 255] for global indices [start, start+count)."""
    base = (seed * _G1 + tensor_id * _G2 + start) & _M64
    idx = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = idx + np.uint64(base)
        z = _splitmix64(z)
    return (z >> np.uint64(56)).astype(np.int32)


def draw(seed: int, tensor_id: int, shape, exponent: int, start: int = 0,
         dtype=np.float64) -> np.ndarray:
    """Values (2m-255)/256 * 2**exponent for a contiguous block of global indices."""
    count = int(np.prod(shape)) if len(shape) else 1
    m = draw_codes(seed, tensor_id, start, count)
    v = (2.0 * m - 255.0) * math.ldexp(1.0, exponent - 8)
    return v.astype(dtype).reshape(shape)


def draw_rows(seed: int, tensor_id: int, row_len: int, rows, exponent: int) -> np.ndarray:
    """Selected rows of a row-major tensor with ``row_len`` columns (global row ids)."""
    rows = np.asarray(rows, dtype=np.int64)
    out = np.empty((len(rows), row_len), dtype=np.float64)
    for i, r in enumerate(rows):
        out[i] = draw(seed, tensor_id, (row_len,), exponent, start=int(r) * row_len)
    return out


def to_bf16_bits(v: np.ndarray) -> np.ndarray:
    """bf16 bit patterns of values that are exactly representable (as produced by draw)."""
    f = np.ascontiguousarray(v, dtype=np.float32)
    bits = f.view(np.uint32)
    if np.any(bits & np.uint32(0xFFFF)):
        raise ValueError("value not exactly representable in bf16")
    return (bits >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    """fp64 values of bf16 bit patterns (exact)."""
    u = (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16))
    return u.view(np.float32).astype(np.float64)


def exponent_for_std(std: float) -> int:
    """Power-of-two range 2^e whose uniform std (2^e/sqrt(3)) is closest to ``std``."""
    return int(round(math.log2(std * math.sqrt(3.0))))


def layer_exponents(D: int, Hq: int, d: int, S: int, profile: str = "benign") -> dict:
    """Exponents for the layer inputs.

    benign: x std~1, Wq/Wk/Wv std~1/sqrt(D), Wo std~1/sqrt(Hq*d), dY std~1/sqrt(S)
            -> attention scores with std ~ 1.
    peaky:  Wq/Wk twice as large (score std ~ 4); reported, not gated.
    """
    e = {
        "x": exponent_for_std(1.0),
        "wq": exponent_for_std(1.0 / math.sqrt(D)),
        "wk": exponent_for_std(1.0 / math.sqrt(D)),
        "wv": exponent_for_std(1.0 / math.sqrt(D)),
        "wo": exponent_for_std(1.0 / math.sqrt(Hq * d)),
        "dy": exponent_for_std(1.0 / math.sqrt(S)),
    }
    # Powers of two cannot hit std 1 exactly: pick Wk's exponent so that the
    # predicted score std  sx^2 * sq * sk * D  (q.k/sqrt(d) with d cancelling) is closest to 1.
    sx = 2.0 ** e["x"] / math.sqrt(3.0)

    def score_std(ewk):
        sq = 2.0 ** e["wq"] / math.sqrt(3.0)
        sk = 2.0 ** ewk / math.sqrt(3.0)
        return sx * sx * sq * sk * D

    e["wk"] = min((e["wq"], e["wq"] - 1, e["wq"] + 1), key=lambda v: abs(math.log(score_std(v))))
    if profile == "peaky":
        e["wq"] += 1
        e["wk"] += 1
    elif profile != "benign":
        raise ValueError(profile)
    return e


def layer_inputs(seed: int, S: int, D: int, Hq: int, Hkv: int, d: int,
                 profile: str = "benign", rows=None) -> dict:
    """All layer inputs in fp64 (exact bf16 values), global token indexing.

    ``rows``: optional (start, stop) token range of X and dY to draw (a sequence shard).
    """
    e = layer_exponents(D, Hq, d, S, profile)
    t0, t1 = (0, S) if rows is None else rows
    return {
        "x": draw(seed, TID["x"], (t1 - t0, D), e["x"], start=t0 * D),
        "wq": draw(seed, TID["wq"], (Hq * d, D), e["wq"]),
        "wk": draw(seed, TID["wk"], (Hkv * d, D), e["wk"]),
        "wv": draw(seed, TID["wv"], (Hkv * d, D), e["wv"]),
        "wo": draw(seed, TID["wo"], (D, Hq * d), e["wo"]),
        "dy": draw(seed, TID["dy"], (t1 - t0, D), e["dy"], start=t0 * D),
        "exponents": e,
    }


def core_inputs(seed: int, S: int, Hq: int, Hkv: int, d: int, score_std: float = 1.0) -> dict:
    """Attention-core inputs Q[S,Hq,d], K/V[S,Hkv,d], dO[S,Hq,d] (fp64 exact bf16 values).

    Q and K get std ~ (score_std * sqrt(d))**0.5 / d**0.25 so that q.k/sqrt(d) has std ~ score_std.
    """
    eq = exponent_for_std(math.sqrt(score_std))
    return {
        "q": draw(seed, TID["q"], (S, Hq, d), eq),
        "k": draw(seed, TID["k"], (S, Hkv, d), eq),
        "v": draw(seed, TID["v"], (S, Hkv, d), 0),
        "do": draw(seed, TID["do"], (S, Hq, d), 0),
        "exponents": {"q": eq, "k": eq, "v": 0, "do": 0},
    }


def payload_bits(seed: int, tensor_id: int, shape, start: int = 0) -> np.ndarray:
    """Index payloads for the bit-exact layout tests: a bf16 bit pattern per global element index,
    finite and normal (sign from the hash, biased exponent in [112, 143], 7 hashed mantissa bits:
    8192 distinct values), so a misplaced element is caught with probability ~1 - 1/8192 each.
    Values pass unchanged through a copy, a one-hot projection (x * 1 + zeros) or an all-to-all."""
    count = int(np.prod(shape)) if len(shape) else 1
    base = (seed * _G1 + tensor_id * _G2 + start) & _M64
    with np.errstate(over="ignore"):
        z = _splitmix64(np.arange(count, dtype=np.uint64) + np.uint64(base))
    sign = (z >> np.uint64(63)) << np.uint64(15)
    expo = (np.uint64(112) + ((z >> np.uint64(40)) & np.uint64(31))) << np.uint64(7)
    mant = (z >> np.uint64(20)) & np.uint64(0x7F)
    return (sign | expo | mant).astype(np.uint16).reshape(shape)


def norm_weight(seed: int, name: str, d: int) -> np.ndarray:
    """Qwen3 q/k RMSNorm weight vector [d]: 1 + k/128, k = m mod 33 - 16 in [-16, 16]
    (values 0.875 .. 1.125 around the trained weights' typical 1; exact in bf16: spacing 2^-7 in [1, 2),
    2^-8 in [0.5, 1))."""
    m = draw_codes(seed, TID[name], 0, d)
    return 1.0 + ((m % 33) - 16).astype(np.float64) / 128.0
