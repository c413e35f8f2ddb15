"""Shared test helpers (fixture fiber A of tests/golden/spec_examples.jsonl)."""
import numpy as np
import pytest


def fiber_A() -> np.ndarray:
    """The fixed non-palindromic fiber 'A' of tests/golden/spec_examples.jsonl.

    Dyadic coordinates (exact in FP32 and double): a_i = (2i-20, i^2/8, (i mod 3)/2).
    """
    i = np.arange(21, dtype=np.float64)
    return np.stack([2 * i - 20, i * i / 8.0, (i % 3) / 2.0], axis=1).astype(np.float32)


def parse_fiber(expr: str) -> np.ndarray:
    """'A', 'reverse(A)', 'A+(x,y,z)' -> float32 [21,3]."""
    a = fiber_A()
    if expr == "A":
        return a
    if expr == "reverse(A)":
        return np.ascontiguousarray(a[::-1])
    if expr.startswith("A+(") and expr.endswith(")"):
        t = np.array([float(v) for v in expr[3:-1].split(",")], dtype=np.float32)
        return (a + t[None, :]).astype(np.float32)
    raise ValueError(expr)


@pytest.fixture
def A():
    return fiber_A()
