"""Seeded synthetic instances with the shapes / distributions of BASELINE.json's
configs (the reference measures on synthetic data only: PAPER.md:930-933;
no dataset exists to download). numpy PCG64 streams; the seed is recorded in
every bench line.

    c1  dense 500 x 2000,  50-sparse, noise sigma 0.01,   lam = 0.5 lam_max
    c2  dense 2500 x 10000, 250-sparse, 30 dB SNR,         lam = 0.2 lam_max
    c3  Kronecker sum 4096 x 16384 (6 terms of 64x128 factors, 2^-r weights,
        column-normalised), approximations = first {1,2,4} terms with exact
        per-atom errors, 400-sparse, 30 dB SNR, lam = 0.3 lam_max
    c4  dense 8192 x 65536, 800-sparse, 20 dB SNR, 10-point lam path 0.9 -> 0.05
    c5  dense 1024 x 4096, 512 signals x 40-sparse, 30 dB, lam_b = 0.25 lam_max_b
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

CONFIGS = {
    "c1": dict(n=500, k=2000, nnz=50, sigma=0.01, snr_db=None, lam_ratio=0.5),
    "c2": dict(n=2500, k=10000, nnz=250, sigma=None, snr_db=30.0, lam_ratio=0.2),
    "c3": dict(m=64, q=128, terms=6, levels=(1, 2, 4), nnz=400, sigma=None, snr_db=30.0, lam_ratio=0.3),
    "c4": dict(n=8192, k=65536, nnz=800, sigma=None, snr_db=20.0,
               lam_ratios=tuple(0.9 * (0.05 / 0.9) ** (i / 9) for i in range(10))),
    "c5": dict(n=1024, k=4096, nnz=40, batch=512, sigma=None, snr_db=30.0, lam_ratio=0.25),
}


@dataclasses.dataclass
class DenseInstance:
    a: np.ndarray        # N x K, Fortran order, unit-norm columns
    x0: np.ndarray
    y: np.ndarray
    lam_max: float
    lam: float
    seed: int


def gaussian_dictionary(rng: np.random.Generator, n: int, k: int) -> np.ndarray:
    """iid N(0,1) drawn column by column, columns normalised to unit l2."""
    at = rng.standard_normal((k, n))  # row j = column j
    at /= np.sqrt(np.einsum("ij,ij->i", at, at))[:, None]
    return at.T  # Fortran-ordered N x K view


def sparse_signal(rng: np.random.Generator, k: int, nnz: int) -> np.ndarray:
    x0 = np.zeros(k)
    pos = rng.choice(k, size=nnz, replace=False)
    x0[pos] = rng.standard_normal(nnz)
    return x0


def observe(rng: np.random.Generator, clean: np.ndarray, sigma: Optional[float], snr_db: Optional[float]) -> np.ndarray:
    n = clean.size
    if sigma is None:
        sigma = np.linalg.norm(clean) / np.sqrt(n) * 10.0 ** (-snr_db / 20.0)
    return clean + sigma * rng.standard_normal(n)


def dense_instance(name: str, seed: Optional[int] = None, n: Optional[int] = None, k: Optional[int] = None,
                   nnz: Optional[int] = None) -> DenseInstance:
    cfg = dict(CONFIGS[name])
    seed = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}[name] if seed is None else seed
    n = n or cfg["n"]
    k = k or cfg["k"]
    nnz = nnz or cfg["nnz"]
    rng = np.random.default_rng(seed)
    a = gaussian_dictionary(rng, n, k)
    x0 = sparse_signal(rng, k, nnz)
    y = observe(rng, a @ x0, cfg.get("sigma"), cfg.get("snr_db"))
    lam_max = float(np.max(np.abs(a.T @ y)))
    lam = cfg.get("lam_ratio", 1.0) * lam_max
    return DenseInstance(a=a, x0=x0, y=y, lam_max=lam_max, lam=lam, seed=seed)


@dataclasses.dataclass
class SukroInstance:
    lefts: list          # B_t (m x q), 2^-t weight folded in
    rights: list         # C_t (m x q)
    col_scale: np.ndarray
    a: np.ndarray        # exact dense N x K (column-normalised sum)
    levels: tuple        # number of terms per approximate level
    eps: list            # per level, running max finer -> coarser (dictionary.cpp:344-349)
    approx_norms: list
    exact_norms: np.ndarray
    rc: list
    x0: np.ndarray
    y: np.ndarray
    lam_max: float
    lam: float
    seed: int


def kron_dense(lefts, rights, col_scale=None) -> np.ndarray:
    """Explicit sum_t B_t (x) C_t (column j = jb*q + jc, row i = rb*m + rc)."""
    a = sum(np.kron(b, c) for b, c in zip(lefts, rights))
    if col_scale is not None:
        a = a * col_scale[None, :]
    return np.asfortranarray(a)


def sukro_instance(seed: int = 3, m: int = 64, q: int = 128, terms: int = 6, levels=(1, 2, 4), nnz: int = 400,
                   snr_db: float = 30.0, lam_ratio: float = 0.3) -> SukroInstance:
    rng = np.random.default_rng(seed)
    lefts, rights = [], []
    for r in range(1, terms + 1):
        lefts.append(2.0 ** (-r) * rng.standard_normal((m, q)))
        rights.append(rng.standard_normal((m, q)))
    raw = kron_dense(lefts, rights)
    norms = np.sqrt(np.einsum("ij,ij->j", raw, raw))
    scale = 1.0 / norms
    a = np.asfortranarray(raw * scale[None, :])
    exact_norms = np.sqrt(np.einsum("ij,ij->j", a, a))
    eps, an, rc = [], [], []
    n, k = m * m, q * q
    for nt in levels:
        approx = kron_dense(lefts[:nt], rights[:nt], scale)
        eps.append(np.sqrt(np.einsum("ij,ij->j", a - approx, a - approx)))
        an.append(np.sqrt(np.einsum("ij,ij->j", approx, approx)))
        rc.append(nt * (m * k + q * n) / (n * k))  # dictionary.cpp:179-185 / N K
    for i in range(len(eps) - 1, 0, -1):  # running max finer -> coarser
        eps[i - 1] = np.maximum(eps[i - 1], eps[i])
    x0 = sparse_signal(rng, k, nnz)
    y = observe(rng, a @ x0, None, snr_db)
    lam_max = float(np.max(np.abs(a.T @ y)))
    return SukroInstance(lefts=lefts, rights=rights, col_scale=scale, a=a, levels=tuple(levels), eps=eps,
                         approx_norms=an, exact_norms=exact_norms, rc=rc, x0=x0, y=y, lam_max=lam_max,
                         lam=lam_ratio * lam_max, seed=seed)


def sukro_sequence(inst: SukroInstance, backend=None):
    """The configs[2] ApproxSequence: SuKro truncations to the first q in inst.levels
    terms (same column scale, exact per-atom error norms) followed by the exact dense
    dictionary (dictionary.cpp:216-251 invariants)."""
    from . import fastl1 as F

    levels = []
    for li, nt in enumerate(inst.levels):
        op = F.SukroDictionary(list(zip(inst.lefts[:nt], inst.rights[:nt])), col_scale=inst.col_scale,
                               backend=backend)
        levels.append(F.ApproxDictionary(op, inst.eps[li], float(inst.eps[li].max()), inst.rc[li],
                                         inst.approx_norms[li], inst.exact_norms))
    levels.append(F.make_exact_approx(F.DenseDictionary(inst.a, backend=backend)))
    return F.ApproxSequence(levels)
