"""Shared helpers for the parity tests (test infrastructure; imports oracle/)."""
from __future__ import annotations

import functools

import numpy as np

from oracle.oracle import Oracle, Reference  # the checkers (test-only)

TOL = {np.dtype(np.float32): 1e-5, np.dtype(np.float64): 1e-12}  # tests/test_util.hpp:110-113


@functools.lru_cache(maxsize=None)
def oracle() -> Oracle:
    return Oracle()


@functools.lru_cache(maxsize=None)
def reference():
    try:
        return Reference()
    except FileNotFoundError:
        return None


def rel_err_inf(got, want) -> float:
    return Oracle.rel_err_inf(got, want)


def bits(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view(np.uint32 if a.dtype == np.float32 else np.uint64)


def mismatches(a, b) -> int:
    return int((bits(a) != bits(b)).sum())


def fused_sizes(dtype) -> set:
    """Sizes at which the reference's g++ -O3 -march=native code is a strict
    FMA chain (re-verified by tests/test_oracle.py)."""
    if np.dtype(dtype) == np.float32:
        return {1, 5, 6, 7} | set(range(9, 17))
    return {1} | set(range(5, 17))


def rng(seed: int):
    return np.random.default_rng(seed)


def uniform(g, n, dtype):
    return (g.random(n) * 2 - 1).astype(dtype)


def ints(g, n, dtype):
    return g.integers(-3, 4, n).astype(dtype)


def to_dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def to_host(t):
    return t.cpu().numpy()
