"""Seeded synthetic inputs for the SMILE layer -- shared by tests/, bench.py and smoke().

This module holds NO arithmetic of the method (no routing, softmax, capacity, FFN or
loss): it only draws random numbers and rounds them to the storage dtype.  Both the CPU
oracle (``oracle/``) and the CUDA path (``paper_2212_05191_b200``) receive its arrays as
inputs, so neither side generates data for the other.

Recipe:
  * x ~ N(0, 1) per rank, rounded to the layer dtype.
  * router W = [W_p; W_q] ~ U(+-1/sqrt(d)) (balanced routing, logit std ~0.58).
  * supplied logits: "balanced" N(0, 0.58); "skewed" N(0, 1) - ln(k+1) (Zipf-like
    popularity, exercises drops); "ties" drawn from {-1, 0, 1} (plants exact ties); "signed_zero" from {-1, -0.0, +0.0, 1}
    (R28: signed-zero ties).
  * experts: W1 ~ U(+-1/sqrt(d)), W2 ~ U(+-1/sqrt(d_ff)); biases 0 for the bench,
    U(+-0.1) for parity runs.
Seeds: stream (seed, rank, tag) through numpy's SeedSequence, so every rank's inputs are
independent of how many ranks are generated.
"""
from __future__ import annotations

import numpy as np

_TAGS = {"x": 1, "logits": 2, "router": 3, "w1": 4, "b1": 5, "w2": 6, "b2": 7, "grad": 8}


def rng(seed: int, rank: int, tag: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, rank, _TAGS[tag]])))


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returned as fp32."""
    a = np.ascontiguousarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def to_dtype(a: np.ndarray, dtype: str) -> np.ndarray:
    return round_bf16(a) if dtype == "bf16" else np.ascontiguousarray(a, np.float32)


def tokens(G: int, T: int, d: int, seed: int = 0, dtype: str = "fp32") -> np.ndarray:
    """x [G, T, d]: N(0, 1) per rank."""
    out = np.empty((G, T, d), np.float32)
    for r in range(G):
        out[r] = rng(seed, r, "x").standard_normal((T, d), dtype=np.float32)
    return to_dtype(out, dtype)


def supplied_logits(G: int, T: int, K: int, seed: int = 0, dist: str = "balanced",
                    K1: int | None = None) -> np.ndarray:
    """Router logits [G, T, K] fp32.  For 'skewed' the popularity bias restarts at each
    level boundary K1 so both levels are skewed."""
    out = np.empty((G, T, K), np.float32)
    for r in range(G):
        g = rng(seed, r, "logits")
        if dist == "balanced":
            out[r] = 0.58 * g.standard_normal((T, K), dtype=np.float32)
        elif dist == "skewed":
            k = np.arange(K)
            if K1 is not None:
                k = np.where(k < K1, k, k - K1)
            out[r] = g.standard_normal((T, K), dtype=np.float32) - np.log1p(k).astype(np.float32)
        elif dist == "ties":
            out[r] = g.integers(-1, 2, size=(T, K)).astype(np.float32)
        elif dist == "signed_zero":
            # R28: entries from {-1, -0.0, +0.0, +1} -- -0.0 and +0.0 compare equal under '>',
            # so a row whose maxima are signed zeros is a tie the lowest index wins
            v = g.integers(-1, 2, size=(T, K)).astype(np.float32)
            neg = g.integers(0, 2, size=(T, K)).astype(bool)
            out[r] = np.where((v == 0) & neg, np.float32(-0.0), v)
        else:
            raise ValueError(dist)
    return out


def router_weights(K: int, d: int, seed: int = 0) -> np.ndarray:
    """Tied router W [K, d] ~ U(+-1/sqrt d) (rows 0..K1-1 = W_p, the rest = W_q)."""
    b = 1.0 / np.sqrt(d)
    return rng(seed, 0, "router").uniform(-b, b, size=(K, d)).astype(np.float32)


def expert_weights(NE: int, d: int, d_ff: int, seed: int = 0, dtype: str = "fp32",
                   bias: bool = True):
    """Expert bank indexed by global expert id: W1 [NE, d, d_ff], b1 [NE, d_ff],
    W2 [NE, d_ff, d], b2 [NE, d] (the FFN of SPEC's expert module)."""
    b1w, b2w = 1.0 / np.sqrt(d), 1.0 / np.sqrt(d_ff)
    W1 = np.empty((NE, d, d_ff), np.float32)
    W2 = np.empty((NE, d_ff, d), np.float32)
    b1 = np.zeros((NE, d_ff), np.float32)
    b2 = np.zeros((NE, d), np.float32)
    for g in range(NE):
        W1[g] = rng(seed, g, "w1").uniform(-b1w, b1w, size=(d, d_ff))
        W2[g] = rng(seed, g, "w2").uniform(-b2w, b2w, size=(d_ff, d))
        if bias:
            b1[g] = rng(seed, g, "b1").uniform(-0.1, 0.1, size=d_ff)
            b2[g] = rng(seed, g, "b2").uniform(-0.1, 0.1, size=d)
    return tuple(to_dtype(a, dtype) for a in (W1, b1, W2, b2))
