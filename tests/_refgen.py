"""Test-only restatements of the reference's instance generators and test oracles.

Follows, line by line:
  tests/helpers.hpp:35-89     random_matrix / random_vector / random_dictionary / random_instance
  tests/helpers.hpp:101-179   solve_oracle (FISTA + LDL^T support polishing + KKT check)
  test_fastl1.cpp:18-39     square_instance / degenerate_sequence
  dictionary.cpp:37-45, 253-357, 384-434
                              rearrange, truncated_svd, build_sukro_sequence, synthesize_scenario
The mt19937_64 / std::normal_distribution streams come from the oracle library
(orc_gen_normals / orc_gen_support, libstdc++), so matrices are the reference's
own bytes; QR / SVD use LAPACK through numpy (Householder sign conventions match
Eigen's; singular-vector sign flips cancel in B (x) C).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np


class RefGen:
    def __init__(self, oracle_backend):
        self.lib = oracle_backend.lib

    # ---- RNG streams
    def normals(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count)
        self.lib.gen_normals(seed & 0xFFFFFFFFFFFFFFFF, count, out.ctypes.data_as(C.POINTER(C.c_double)))
        return out

    def support(self, seed: int, k: int, support: int):
        pos = np.empty(support, dtype=np.int64)
        val = np.empty(support)
        self.lib.gen_support(seed & 0xFFFFFFFFFFFFFFFF, k - 1, support, pos.ctypes.data_as(C.POINTER(C.c_int64)),
                             val.ctypes.data_as(C.POINTER(C.c_double)))
        return pos, val

    # ---- helpers.hpp
    def random_matrix(self, rows: int, cols: int, seed: int) -> np.ndarray:
        return self.normals(seed, rows * cols).reshape(cols, rows).T.copy(order="F")

    def random_vector(self, n: int, seed: int) -> np.ndarray:
        return self.normals(seed ^ 0xABCDEF, n)

    def random_dictionary(self, n: int, k: int, seed: int) -> np.ndarray:
        m = self.random_matrix(n, k, seed)
        return np.asfortranarray(m / np.linalg.norm(m, axis=0)[None, :])

    def random_instance(self, n, k, ratio, seed, support=5):
        a = self.random_dictionary(n, k, seed)
        pos, val = self.support(seed ^ 0x5117, k, support)
        x = np.zeros(k)
        for p, v in zip(pos, val):
            x[p] = v
        y = a @ x
        y = y / np.linalg.norm(y)
        lmax = float(np.max(np.abs(a.T @ y)))
        return a, y, ratio * lmax, lmax

    # ---- dictionary.cpp
    def synthesize_scenario(self, n: int, k: int, scenario: str, seed: int) -> np.ndarray:
        m, q = _isqrt(n), _isqrt(k)
        n_terms = min(40, m)
        ratio = {"easy": 0.3, "moderate": 0.6, "hard": 0.95}[scenario]
        # one shared stream: seed ^ 0xd1c7, consumed by 2*q random_frame calls in order
        stream = self.normals(seed ^ 0xD1C7, 2 * q * m * n_terms)
        off = 0

        def frame():
            nonlocal off
            g = stream[off:off + m * n_terms].reshape(n_terms, m).T
            off += m * n_terms
            qm, _ = np.linalg.qr(g, mode="reduced")
            return qm

        left = [np.zeros((m, q)) for _ in range(n_terms)]
        right = [np.zeros((m, q)) for _ in range(n_terms)]
        col_scale = 1.0 / np.sqrt(q)
        for j in range(q):
            fb = frame()
            fc = frame()
            for t in range(n_terms):
                left[t][:, j] = col_scale * fb[:, t]
                right[t][:, j] = col_scale * fc[:, t]
        a = np.zeros((n, k))
        for t in range(n_terms):
            sv = ratio ** t
            a += np.kron(sv * left[t], right[t])
        norms = np.linalg.norm(a, axis=0)
        return np.asfortranarray(a / norms[None, :])

    def truncated_svd(self, mat: np.ndarray, rank: int):
        mindim = min(mat.shape)
        p = min(rank + 8, mindim)
        omega = self.normals(0x5EEDF00D, mat.shape[1] * p).reshape(p, mat.shape[1]).T
        y = mat @ omega

        def orth(a):
            return np.linalg.qr(a, mode="reduced")[0]

        for _ in range(6):
            qm = orth(y)
            y = mat @ (mat.T @ qm)
        qm = orth(y)
        bt = mat.T @ qm
        U, s, Vt = np.linalg.svd(bt, full_matrices=False)
        u = qm @ Vt.T[:, :rank]
        v = U[:, :rank]
        return u, s[:rank], v

    def build_sukro_sequence(self, a: np.ndarray, ranks):
        """-> list of dicts (terms, eps, op_err, rc, approx_norms, exact_norms) + exact."""
        n, k = a.shape
        m, q = _isqrt(n), _isqrt(k)
        # rearrange: R(i + j*m, rr + s*m) = A(i*m + rr, j*q + s)
        R = a.reshape(m, m, q, q, order="F")  # A[rr + i*m, s + j*q] -> R4[rr, i, s, j]
        R = R.transpose(1, 3, 0, 2).reshape(m * q, m * q, order="F")  # rows i + j*m, cols rr + s*m
        u, s, v = self.truncated_svd(R, max(ranks))
        terms = []
        for t in range(max(ranks)):
            sc = np.sqrt(max(s[t], 0.0))
            terms.append((u[:, t].reshape(m, q, order="F") * sc, v[:, t].reshape(m, q, order="F") * sc))
        exact_norms = np.linalg.norm(a, axis=0)
        levels = []
        residual = a.copy()
        dense_flops = n * k
        nxt = 0
        for t in range(max(ranks)):
            residual -= np.kron(terms[t][0], terms[t][1])
            if t + 1 == ranks[nxt]:
                nt = ranks[nxt]
                mv = nt * (m * k + q * n)
                levels.append(dict(terms=terms[:nt], eps=np.linalg.norm(residual, axis=0),
                                   approx_norms=np.linalg.norm(a - residual, axis=0), rc=mv / dense_flops))
                nxt += 1
                if nxt == len(ranks):
                    break
        for i in range(len(levels) - 1, 0, -1):
            levels[i - 1]["eps"] = np.maximum(levels[i - 1]["eps"], levels[i]["eps"])
        for lv in levels:
            lv["op_err"] = float(lv["eps"].max())
            lv["exact_norms"] = exact_norms
        return levels

    def square_instance(self, n, k, seed, support=4, scenario="moderate"):
        a = self.synthesize_scenario(n, k, scenario, seed)
        pos, val = self.support(seed ^ 0x99, k, support)
        x = np.zeros(k)
        for p_, v_ in zip(pos, val):
            x[p_] = v_
        y = a @ x
        y = y / np.linalg.norm(y)
        lmax = float(np.max(np.abs(a.T @ y)))
        return a, y, lmax


def _isqrt(v: int) -> int:
    r = int(round(v ** 0.5))
    while r * r > v:
        r -= 1
    while (r + 1) * (r + 1) <= v:
        r += 1
    if r * r != v:
        raise ValueError(f"{v} must be a perfect square")
    return r


def make_sequence(F, backend, a, levels=None):
    """ApproxSequence from build_sukro_sequence output (or just the exact dictionary)."""
    out = []
    for lv in levels or []:
        op = F.SukroDictionary(lv["terms"], backend=backend)
        out.append(F.ApproxDictionary(op, lv["eps"], lv["op_err"], lv["rc"], lv["approx_norms"], lv["exact_norms"]))
    out.append(F.make_exact_approx(F.DenseDictionary(a, backend=backend)))
    return F.ApproxSequence(out)


def perturbed_approx(F, backend, rg: RefGen, exact: np.ndarray, noise: float, seed: int, rc: float = 0.5):
    """test_screening.cpp:24-39: a dense 'approximation' A + noise*G with measured eps."""
    approx = exact + noise * rg.random_matrix(exact.shape[0], exact.shape[1], seed)
    eps = np.linalg.norm(approx - exact, axis=0)
    op = F.DenseDictionary(approx, backend=backend)
    return F.ApproxDictionary(op, eps, float(eps.max()), rc, np.linalg.norm(approx, axis=0),
                              np.linalg.norm(exact, axis=0)), approx


@dataclass
class OracleSolution:
    x: np.ndarray
    theta: np.ndarray
    gap: float


def soft(z, u):
    mag = np.abs(z) - u
    return np.where(mag <= 0.0, 0.0, np.sign(z) * mag)


def solve_oracle(a: np.ndarray, y: np.ndarray, lam: float, target_gap: float = 1e-12,
                 max_iter: int = 400000) -> OracleSolution:
    """helpers.hpp:101-179 restated with numpy (independent of both libraries)."""
    k = a.shape[1]
    l = np.linalg.svd(a, compute_uv=False)[0]
    inv_l = 1.0 / (l * l * 1.0000001)

    def gap_of(x):
        rho = y - a @ x
        corr = a.T @ rho
        infn = np.max(np.abs(corr))
        proj = y @ rho / (lam * max(rho @ rho, 1e-300))
        alpha = 1.0 / infn if infn > 0 else 1e300
        s = min(max(proj, -alpha), alpha)
        theta = s * rho
        primal = 0.5 * rho @ rho + lam * np.abs(x).sum()
        dual = 0.5 * y @ y - 0.5 * lam * lam * np.sum((theta - y / lam) ** 2)
        return primal - dual

    x = np.zeros(k)
    x_prev = x.copy()
    t_k = 1.0
    for it in range(max_iter):
        t_next = 0.5 * (1.0 + np.sqrt(1.0 + 4.0 * t_k * t_k))
        mom = (t_k - 1.0) / t_next
        w = x + mom * (x - x_prev)
        gp = w + inv_l * (a.T @ (y - a @ w))
        x_prev, x = x, soft(gp, lam * inv_l)
        t_k = t_next
        if it % 50 == 49:
            supp = np.nonzero(x)[0]
            if 0 < supp.size < a.shape[0]:
                As = a[:, supp]
                signs = np.sign(x[supp])
                xs = np.linalg.solve(As.T @ As, As.T @ y - lam * signs)
                if np.all(xs * signs >= 0):
                    cand = np.zeros(k)
                    cand[supp] = xs
                    theta = (y - a @ cand) / lam
                    if np.max(np.abs(a.T @ theta)) <= 1.0 + 1e-12 and gap_of(cand) <= target_gap:
                        x = cand
                        break
            if gap_of(x) <= target_gap:
                break
    g = gap_of(x)
    if g > target_gap:
        raise RuntimeError(f"oracle did not reach the target gap: {g}")
    return OracleSolution(x=x, theta=(y - a @ x) / lam, gap=g)
