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


# ------------------------------------------------------------------ device inputs
def device_input(cfg: int, dev, handle=None) -> dict:
    """The config's input generated on the GPU through libqdwhg (seeded device
    Gaussian, our own Householder QR for the orthogonal factors, DMMA GEMMs).
    The generating handle runs in deterministic mode (QDWHG_FLAG_DETERMINISTIC:
    fixed-order panel reductions), so the bytes — and input_sha256() — are the
    same on every run and every B200; the full-size parity fixtures
    (tests/golden/fullsize/) are keyed by that hash."""
    import torch
    from . import qdwh
    c = dict(CONFIGS[cfg])
    h = handle if handle is not None else qdwh.Handle(device=dev.index or 0, deterministic=True)
    if c["kind"] == "eig":
        n = c["n"]
        if c["family"] == "wishart":
            G = qdwh.gaussian_matrix_device(n, n, c["seed"], device=dev, handle=h)
            A = torch.empty((n, n), dtype=torch.float64, device=dev).t()
            qdwh.gemm(G, G, A, alpha=1.0 / n, trans_a=True, handle=h)
            del G
            A -= torch.eye(n, dtype=torch.float64, device=dev)
            A = (0.5 * (A + A.t())).t().contiguous().t()
            return dict(A=A, c=c["shift"], k=c["k"], truth=None, kind="eig", cfg=cfg)
        lam = config_eigenvalues(c["family"], n, c["seed"])
        G = qdwh.gaussian_matrix_device(n, n, c["seed"], device=dev, handle=h)
        Q, _ = qdwh.qr_factor(G, handle=h)
        del G
        QL = (Q * torch.from_numpy(lam).to(dev)[None, :]).t().contiguous().t()
        A = torch.empty((n, n), dtype=torch.float64, device=dev).t()
        qdwh.gemm(QL, Q, A, trans_b=True, handle=h)
        A = (0.5 * (A + A.t())).t().contiguous().t()
        k = c["k"]
        return dict(A=A, c=largest_k_shift(lam, k), k=k, truth=np.sort(lam)[::-1][:k], kind="eig",
                    cfg=cfg)
    m, n = c["m"], c["n"]
    sig = config_singular_values(c["family"], n)
    Gl = qdwh.gaussian_matrix_device(m, n, c["seed"] ^ LEFT_STREAM, device=dev, handle=h)
    U = qdwh.qr_factor(Gl, handle=h)[0][:, :n]  # thin Q (first n columns)
    del Gl
    Gr = qdwh.gaussian_matrix_device(n, n, c["seed"] ^ RIGHT_STREAM, device=dev, handle=h)
    V, _ = qdwh.qr_factor(Gr, handle=h)
    del Gr
    US = (U * torch.from_numpy(sig).to(dev)[None, :]).t().contiguous().t()
    del U
    A = torch.empty((n, m), dtype=torch.float64, device=dev).t()
    qdwh.gemm(US, V, A, trans_b=True, handle=h)
    k = c["k"]
    return dict(A=A, cut=sigma_cut(sig, k), k=k, truth=np.sort(sig)[::-1][:k], kind="svd", cfg=cfg,
                randomize=bool(c.get("randomize", False)))


def host_copy(A) -> np.ndarray:
    """Column-major host copy (numpy, Fortran order) of a device matrix."""
    return np.asfortranarray(A.cpu().numpy())


def input_sha256(a_host: np.ndarray) -> str:
    """SHA-256 of the column-major FP64 bytes (the QDWH-file payload order)."""
    import hashlib
    return hashlib.sha256(np.asfortranarray(a_host).tobytes(order="F")).hexdigest()
