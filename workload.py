"""Seeded synthetic inputs for the hot path — shared by tests, the oracle checks and bench.py.

This module is INPUT SYNTHESIS ONLY. It holds none of the hot path's arithmetic
(no Toeplitz gather, no projection S_l = U* T_l V Sigma^-1, no Vandermonde power
tables, no least-squares products): those live, independently, in ``oracle/``
(CPU reference) and in ``paper_2012_11430_b200/csrc`` (CUDA path). Neither of
those imports the other; both may import this module.

What it synthesizes (recipe also stated in DESIGN.md §3):

* planted parameters t_j in [0,1)^d and coefficients c_j != 0 of the exponential
  sum f(k) = sum_j c_j exp(-2 pi i <t_j,k>)              (eq_exp_sum)
* the sample grid f~(k) = f(k)(1+delta_k) on the box {-n..n+1}^d, lexicographic,
  last coordinate fastest
* the paper's test family t_j(i) = ((i-1)m+j-1) 10^-ceil(log10(dm)), c_j = j+ij
                                                         
* the rank-m SVD inputs U, V, Sigma of the NOISE-FREE T (reading R20): any
  valid reduced SVD is a legal input of eq_generateSl; the planted
  one is obtained without forming T from the factorization T = B diag(c) B^H with
  B[k,j] = exp(-2 pi i <t_j,k>) (a QR of B and an m x m SVD, numpy library calls).
* the node vector z_j = exp(-2 pi i t_j) used as input of the LS step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 201211430


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""
    name: str
    d: int
    n: int
    m: int
    noise: float          # relative complex-Gaussian noise sigma (reading R5)
    seed: int
    note: str = ""

    @property
    def N(self) -> int:
        return (self.n + 1) ** self.d

    @property
    def L(self) -> int:
        return 2 * self.n + 2

    @property
    def box(self) -> int:
        return self.L ** self.d


CONFIGS = {
    "cfg1": Config("cfg1", 2, 10, 3, 0.0, BASE_SEED + 1, "d=2 n=10 N=121 m=3 noise-free"),
    "cfg2": Config("cfg2", 2, 63, 20, 1e-6, BASE_SEED + 2, "d=2 n=63 N=4096 m=20 sigma=1e-6"),
    "cfg3": Config("cfg3", 3, 20, 50, 0.0, BASE_SEED + 3, "d=3 n=20 N=9261 m=50 noise-free"),
    "cfg4": Config("cfg4", 2, 200, 100, 1e-6, BASE_SEED + 4, "d=2 n=200 N=40401 m=100 noisy (headline)"),
    "cfg5": Config("cfg5", 4, 12, 30, 0.0, BASE_SEED + 5, "d=4 n=12 N=28561 m=30 noise-free"),
}


def torus_dist_inf(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Torus infinity-norm distance min(|a-b|, 1-|a-b|) over coordinates (R13)."""
    diff = np.abs(a - b) % 1.0
    return np.max(np.minimum(diff, 1.0 - diff), axis=-1)


def planted_nodes(d: int, m: int, n: int, rng: np.random.Generator) -> np.ndarray:
    """t_j i.i.d. U[0,1)^d, rejection-sampled to torus inf-norm separation >= 2/(n+1)
    (reading R17: the paper's K_d of Thm 2.1, is not given). For tiny test
    grids where that cannot be packed, the separation is capped at 0.5 m^(-1/d)."""
    sep = min(2.0 / (n + 1), 0.5 * m ** (-1.0 / d))
    t = np.empty((m, d))
    cnt = 0
    tries = 0
    while cnt < m:
        cand = rng.random(d)
        tries += 1
        if tries > 1000000:
            raise RuntimeError("could not place separated nodes")
        if cnt == 0 or np.min(torus_dist_inf(t[:cnt], cand[None, :])) >= sep:
            t[cnt] = cand
            cnt += 1
    return t


def planted_coeffs(m: int, rng: np.random.Generator) -> np.ndarray:
    """c_j = (1+u_j) exp(2 pi i phi_j), u, phi ~ U[0,1): |c_j| in [1,2), never 0."""
    u = rng.random(m)
    phi = rng.random(m)
    return (1.0 + u) * np.exp(2j * np.pi * phi)


def paper_family(d: int, m: int):
    """t_j(i) = ((i-1)m + j-1) 10^-ceil(log10(d m)), c_j = j + i j."""
    scale = 10.0 ** (-math.ceil(math.log10(d * m))) if d * m > 1 else 1.0
    t = np.empty((m, d))
    for j in range(1, m + 1):
        for i in range(1, d + 1):
            t[j - 1, i - 1] = ((i - 1) * m + j - 1) * scale
    c = np.array([j + 1j * j for j in range(1, m + 1)], dtype=np.complex128)
    return t, c


def box_coords(d: int, n: int) -> np.ndarray:
    """All k in {-n..n+1}^d, lexicographic, last coordinate fastest; shape (L^d, d)."""
    axis = np.arange(-n, n + 2, dtype=np.int64)
    grids = np.meshgrid(*([axis] * d), indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1)


def index_set(d: int, n: int) -> np.ndarray:
    """I_n = {0..n}^d, lexicographic, last coordinate fastest (reading R2)."""
    axis = np.arange(0, n + 1, dtype=np.int64)
    grids = np.meshgrid(*([axis] * d), indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1)


def evaluate(t: np.ndarray, c: np.ndarray, k: np.ndarray) -> np.ndarray:
    """f(k) = sum_j c_j exp(-2 pi i frac(<t_j,k>)) for a batch of integer points k (P, d).
    The phase <t_j,k> is reduced mod 1 before exponentiation."""
    k = np.atleast_2d(k).astype(np.float64)
    out = np.zeros(k.shape[0], dtype=np.complex128)
    chunk = 1 << 16
    for s in range(0, k.shape[0], chunk):
        ph = k[s:s + chunk] @ t.T                  # (P, m)
        ph = ph - np.floor(ph)
        out[s:s + chunk] = np.exp(-2j * np.pi * ph) @ c
    return out


def noise_pattern(shape, seed: int) -> np.ndarray:
    """One normalized complex Gaussian pattern (xi + i eta)/sqrt(2), E|delta|^2 = 1
    (reading R5; scaled by sigma by the caller)."""
    rng = np.random.default_rng([seed, 7])
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / math.sqrt(2.0)


def disk_pattern(shape, seed: int) -> np.ndarray:
    """One normalized bounded pattern rho e^{i theta}, rho ~ U[0,1], theta ~ U[0, 2 pi): |delta| <= 1
    (the paper's noise model |delta_k| <= eps; reading R5b: SPEC S:73 draws r uniform on
    [0, eps], and the identical mantissas of the table rows 1e-9 / 1e-6, say one pattern is
    reused and scaled by eps)."""
    rng = np.random.default_rng([seed, 13])
    rho = rng.random(shape)
    theta = 2.0 * np.pi * rng.random(shape)
    return rho * np.exp(1j * theta)


def sample_grid(t: np.ndarray, c: np.ndarray, n: int, noise: float = 0.0, seed: int = 0,
                noise_model: str = "gauss") -> np.ndarray:
    """f~(k) = f(k)(1 + delta_k) on the box {-n..n+1}^d (reading R1).
    noise_model "gauss": delta = sigma (xi + i eta)/sqrt 2 (BASELINE configs, reading R5);
    "disk": delta = eps rho e^{i theta}, |delta| <= eps (the paper's accuracy experiment, reading R5b)."""
    d = t.shape[1]
    f = evaluate(t, c, box_coords(d, n))
    if noise > 0.0:
        if noise_model == "gauss":
            f = f * (1.0 + noise * noise_pattern(f.shape, seed))
        elif noise_model == "disk":
            f = f * (1.0 + noise * disk_pattern(f.shape, seed))
        else:
            raise ValueError(noise_model)
    return np.ascontiguousarray(f)


def random_mu(d: int, seed: int) -> np.ndarray:
    """mu ~ complex Gaussian, normalized to ||mu||_2 = 1 (the random point of S_C^{d-1}, PAPER.md:56;
    reading R7). A random draw of the method, passed to both the oracle and the device diagonalization."""
    rng = np.random.default_rng([seed, 11])
    mu = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    return mu / math.sqrt(float(np.sum(np.abs(mu) ** 2)))


def gaussian_block(N: int, r: int, seed: int, which: int) -> np.ndarray:
    """Seeded complex Gaussian N x r block: the random starting matrices U_0 (which=0), V_0 (which=1) of
    Algorithm 3 before orthonormalization (PAPER.md:181 leaves them unspecified; reading R14)."""
    rng = np.random.default_rng([seed, 17, which])
    return np.ascontiguousarray(rng.standard_normal((N, r)) + 1j * rng.standard_normal((N, r)))


def node_vectors(t: np.ndarray) -> np.ndarray:
    """z_j = exp(-2 pi i t_j), shape (m, d)."""
    return np.exp(-2j * np.pi * t)


def planted_svd(t: np.ndarray, c: np.ndarray, n: int):
    """Rank-m reduced SVD T = U Sigma V* of the noise-free T = [f(k-h)] (eq_T_svd,
    PAPER.md:22-26), synthesized from T = B diag(c) B^H, B[k,j] = exp(-2 pi i <t_j,k>)
    (k in I_n), which holds because f(k-h) = sum_j c_j z_j^k conj(z_j^h) for |z_j| = 1.
    QR B = QR, then M = R diag(c) R^H = Us S Vs^H, U = Q Us, V = Q Vs.
    Returns U, V (N x m complex128, C-contiguous) and sigma (m,), nonincreasing."""
    d = t.shape[1]
    k = index_set(d, n).astype(np.float64)
    ph = k @ t.T
    ph = ph - np.floor(ph)
    B = np.exp(-2j * np.pi * ph)                    # (N, m)
    Q, R = np.linalg.qr(B)
    M = (R * c[None, :]) @ R.conj().T
    Us, s, Vh = np.linalg.svd(M)
    U = np.ascontiguousarray(Q @ Us)
    V = np.ascontiguousarray(Q @ Vh.conj().T)
    return U, V, np.ascontiguousarray(s)


def random_orthonormal(N: int, m: int, rng: np.random.Generator) -> np.ndarray:
    """A random N x m matrix with orthonormal columns (for gauge/any-input tests)."""
    X = rng.standard_normal((N, m)) + 1j * rng.standard_normal((N, m))
    Q, _ = np.linalg.qr(X)
    return np.ascontiguousarray(Q)


@dataclass
class Problem:
    """Every array the hot path consumes, for one configuration."""
    cfg: Config
    t: np.ndarray          # (m, d) planted parameters
    c: np.ndarray          # (m,) planted coefficients
    grid: np.ndarray       # (L^d,) complex128 samples on the box
    U: np.ndarray          # (N, m)
    V: np.ndarray          # (N, m)
    sigma: np.ndarray      # (m,)
    z: np.ndarray          # (m, d) nodes for the LS step
    extra: dict = field(default_factory=dict)


def make_problem(cfg: Config | str, with_svd: bool = True) -> Problem:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    rng = np.random.default_rng(cfg.seed)
    t = planted_nodes(cfg.d, cfg.m, cfg.n, rng)
    c = planted_coeffs(cfg.m, rng)
    grid = sample_grid(t, c, cfg.n, cfg.noise, cfg.seed)
    if with_svd:
        U, V, s = planted_svd(t, c, cfg.n)
    else:
        U = V = s = None
    return Problem(cfg, t, c, grid, U, V, s, node_vectors(t))


def custom_config(d: int, n: int, m: int, noise: float = 0.0, seed: int = 12345) -> Config:
    return Config(f"custom_d{d}_n{n}_m{m}", d, n, m, noise, seed)
