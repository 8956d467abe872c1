"""Halton low-dispersion sequence (§4.2 "deterministic,
low-dispersion Halton sequence"; SPEC.md S:119-127 radical inverse).

Input generation only: the library takes samples as an argument
(BASELINE.json north_star ``mpap_build_roadmap(samples, ...)``).
"""
import numpy as np

PRIMES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29)


def halton(index: int, base: int) -> float:
    """Radical inverse of ``index`` (>= 1) in ``base``: halton(1,2)=0.5,
    halton(2,2)=0.25, halton(1,3)=1/3."""
    if index < 1:
        raise ValueError("Halton index starts at 1")
    f = 1.0
    r = 0.0
    i = index
    while i > 0:
        f /= base
        r += f * (i % base)
        i //= base
    return r


def halton_points(start: int, count: int, dims: int) -> np.ndarray:
    """Rows ``start .. start+count-1`` of the Halton sequence in the first
    ``dims`` prime bases, in (0, 1)^dims, float64.  Vectorised form of
    :func:`halton` with the same operation order (identical bits)."""
    if start < 1:
        raise ValueError("Halton index starts at 1")
    idx0 = np.arange(start, start + count, dtype=np.int64)
    out = np.empty((count, dims), dtype=np.float64)
    for j in range(dims):
        b = PRIMES[j]
        i = idx0.copy()
        f = 1.0
        r = np.zeros(count, dtype=np.float64)
        while np.any(i > 0):
            f /= b
            r += f * (i % b).astype(np.float64)
            i //= b
        out[:, j] = r
    return out
