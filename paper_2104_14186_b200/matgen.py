"""Synthetic inputs for the five BASELINE configs (harness, not the product path).

BASELINE.json fixes the spectra families but not every draw; they are pinned
here:

  cfg1  n=1024  lambda_i = 2*to_unit(hash64(seed ^ LAMBDA_STREAM, i)) - 1   (uniform on (-1,1])
  cfg2  n=4096  |lambda_i| = 10^(-8 + 8 i/(n-1)), sign = top bit of hash64(seed ^ SIGN_STREAM, i)
  cfg3  8192^2  sigma_i = 10^(-16 i/(n-1))
  cfg4  n=16384 A = G^T G / n - I (Wishart), G ~ N(0,1) seeded
  cfg5  32768x8192  sigma_i = 1/(i+1)

Orthogonal factors are Q of the Householder QR of seeded Gaussians
(reference pattern matgen.cpp:17-19); left/right factor streams use the
reference's own XOR constants (matgen.cpp:13-15).  hash64/to_unit restate
kernels.cpp:16-26 bit-exactly with numpy uint64 arithmetic.
"""
from __future__ import annotations

import numpy as np

LAMBDA_STREAM = 0x6C616D62   # "lamb"
SIGN_STREAM = 0x7369676E     # "sign"
LEFT_STREAM = 0x71316C65     # matgen.cpp:14 kLeftFactorStream
RIGHT_STREAM = 0x71327269    # matgen.cpp:15 kRightFactorStream

CONFIGS = {
    1: dict(kind="eig", n=1024, family="uniform", k=103, seed=42),
    2: dict(kind="eig", n=4096, family="logsigned", k=41, seed=42),
    3: dict(kind="svd", m=8192, n=8192, family="log16", k=410, seed=42),
    4: dict(kind="eig", n=16384, family="wishart", k=3277, seed=42, shift=0.8881 - 0.05),
    # randomized detection for the slow sigma_i = 1/i decay (l 4546 -> ~2.9k,
    # measured 1.44 -> 1.22 s on one B200); the reference's own use_randomization option
    5: dict(kind="svd", m=32768, n=8192, family="inv", k=819, seed=42, randomize=True),
}


def hash64_np(seed: int, counters: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 (kernels.cpp:16-21); exact mod-2^64 arithmetic."""
    with np.errstate(over="ignore"):
        c = counters.astype(np.uint64)
        z = np.uint64(seed & ((1 << 64) - 1)) + (c + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def to_unit_np(h: np.ndarray) -> np.ndarray:
    """kernels.cpp:24-26 — (0,1], exact."""
    return ((h >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53


def gaussian_host(count: int, seed: int) -> np.ndarray:
    """N(0,1) draws 0..count-1 of the reference's counter generator
    (kernels.cpp:28-32): exact u64 hashing, then glibc log/cos via `math`,
    so the values are bit-identical to qdwh::gaussian_matrix(count, 1, seed)."""
    import math
    i = np.arange(count, dtype=np.uint64)
    u1 = to_unit_np(hash64_np(seed, 2 * i))
    u2 = to_unit_np(hash64_np(seed, 2 * i + 1))
    return np.array([math.sqrt(-2.0 * math.log(a)) * math.cos(2.0 * math.pi * b)
                     for a, b in zip(u1.tolist(), u2.tolist())])


def config_eigenvalues(family: str, n: int, seed: int = 42) -> np.ndarray:
    """Planted eigenvalues, index order (not sorted)."""
    i = np.arange(n)
    if family == "uniform":
        return 2.0 * to_unit_np(hash64_np(seed ^ LAMBDA_STREAM, i)) - 1.0
    if family == "logsigned":
        mag = np.power(10.0, -8.0 + 8.0 * i / max(n - 1, 1))
        sign = np.where((hash64_np(seed ^ SIGN_STREAM, i) >> np.uint64(63)) == 1, -1.0, 1.0)
        return mag * sign
    raise ValueError(family)


def config_singular_values(family: str, n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    if family == "log16":
        return np.power(10.0, -16.0 * i / max(n - 1, 1))
    if family == "inv":
        return 1.0 / (i + 1.0)
    raise ValueError(family)


def largest_k_shift(lam: np.ndarray, k: int) -> float:
    """Shift c strictly between the k-th and (k+1)-th largest eigenvalue:
    the k largest eigenpairs of A are the negative ones of B = cI - A."""
    s = np.sort(lam)[::-1]
    return 0.5 * (s[k - 1] + s[k])


def sigma_cut(sig: np.ndarray, k: int) -> float:
    """Absolute cut sigma* = geometric mean of sigma_k and sigma_{k+1} (1-based)."""
    s = np.sort(sig)[::-1]
    return float(np.sqrt(s[k - 1] * s[k]))


def cut_fraction_s(sig: np.ndarray, k: int, alpha: float) -> float:
    """Relative threshold s = sigma*/alpha for the reference's sigma > s*alpha rule."""
    return sigma_cut(sig, k) / alpha
