"""Instance recipes for BASELINE.json configs[0..4] (seed = config index).

Every instance is a separable QP in the paper's form (P):
    min 1/2 x^T Q x + c^T x   s.t.  A x = b,  x >= 0,   Q = diag(q).
A is dense fp64 and stored column-major (numpy order='F'), matching the device layout.

Draw order is fixed and documented per config so both sides (oracle tests and the GPU
path) see bit-identical inputs.  `make_config(idx, m=.., n=.., ell=..)` produces the same
recipe at a reduced size for tests; the default sizes are the BASELINE.json ones.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

CONFIG_NAMES = {
    0: "cfg0_tiny_m100_n400_l20",
    1: "cfg1_lowrank_m2000_n8000_l50",
    2: "cfg2_svm_N50000_d1000_l100",
    3: "cfg3_portfolio_m64_n200000_l64",
    4: "cfg4_large_m50000_n400000_l200",
}

FULL_SIZES = {  # (m, n, ell) per BASELINE.json configs
    0: (100, 400, 20),
    1: (2000, 8000, 50),
    2: (50000, 1000, 100),   # (N samples, d features, ell); n = 2d + 2N variables
    3: (64, 200000, 64),
    4: (50000, 400000, 200),
}


@dataclass
class QPInstance:
    """One seeded QP instance.  `A` is m x n column-major fp64 (dense configs)."""
    name: str
    idx: int
    A: Optional[np.ndarray]          # m x n, order='F' (None for the structured SVM config)
    q: np.ndarray                    # n, diag of Q (>= 0)
    b: np.ndarray                    # m
    c: np.ndarray                    # n
    ell: int
    x0: Optional[np.ndarray] = None  # generator's feasible primal point (if any)
    y0: Optional[np.ndarray] = None
    z0: Optional[np.ndarray] = None
    extra: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.b.shape[0])

    @property
    def n(self) -> int:
        return int(self.c.shape[0])


def gaussian_matrix(rng: np.random.Generator, m: int, n: int, scale: float = 1.0) -> np.ndarray:
    """m x n i.i.d. N(0, scale^2), column-major.  Drawn column by column (column-major order)."""
    G = rng.standard_normal((n, m)).T  # row-major (n, m) draw == column-major (m, n)
    if scale != 1.0:
        G *= scale
    return np.asfortranarray(G)


def _feasible_bc(A, q, x0, y0, z0):
    # b = A x0 ; c = A^T y0 + z0 - q o x0  (BASELINE.json configs[0]: "gives b=A.x0 and c=...")
    b = A @ x0
    c = A.T @ y0 + z0 - q * x0
    return b, c


def make_config(idx: int, m: Optional[int] = None, n: Optional[int] = None,
                ell: Optional[int] = None, seed: Optional[int] = None) -> QPInstance:
    fm, fn, fl = FULL_SIZES[idx]
    m = fm if m is None else int(m)
    n = fn if n is None else int(n)
    ell = fl if ell is None else int(ell)
    seed = idx if seed is None else int(seed)
    rng = np.random.default_rng(seed)
    name = CONFIG_NAMES[idx] if (m, n, ell) == (fm, fn, fl) else f"cfg{idx}_m{m}_n{n}_l{ell}"

    if idx == 0:
        # draw order: A, q, zero-permutation, x0, y0, z0
        A = gaussian_matrix(rng, m, n, 1.0 / np.sqrt(n))          # A_ij ~ N(0, 1/n)
        q = rng.uniform(0.0, 1.0, n)
        q[rng.permutation(n)[: n // 2]] = 0.0                    # exactly floor(n/2) zeros (A22)
        x0 = rng.uniform(0.5, 1.5, n)
        y0 = rng.standard_normal(m)
        z0 = rng.uniform(0.5, 1.5, n)
        b, c = _feasible_bc(A, q, x0, y0, z0)
        return QPInstance(name, idx, A, q, b, c, ell, x0, y0, z0)

    if idx == 4:
        # counter-based, shardable recipe (synth/large.py); the QP uses generator columns [0, n)
        from .large import generate_shard
        if m * n > 2e8:
            raise ValueError("config 4 at this size is generated per shard on the device (synth.large)")
        sh = generate_shard(m, n, 0, n, n_gen=n, seed=seed)
        A = np.asfortranarray(sh.At[:, :m].numpy().T)
        return QPInstance(name, idx, A, sh.q.numpy(), sh.b_part.numpy(), sh.c.numpy(), ell,
                          sh.x0.numpy(), sh.y0.numpy(), sh.z0.numpy())

    if idx == 1:
        # A = W H + s G ; draw order: W, H, G, q, x0, y0, z0
        r, s = 40, 1e-3
        r = min(r, m, n)
        W = gaussian_matrix(rng, m, r)
        H = gaussian_matrix(rng, r, n)
        G = gaussian_matrix(rng, m, n)
        A = np.asfortranarray(W @ H + s * G)
        del G
        q = rng.uniform(1e-3, 1.0, n)
        x0 = rng.uniform(0.5, 1.5, n)
        y0 = rng.standard_normal(m)
        z0 = rng.uniform(0.5, 1.5, n)
        b, c = _feasible_bc(A, q, x0, y0, z0)
        return QPInstance(name, idx, A, q, b, c, ell, x0, y0, z0)

    if idx == 3:
        # portfolio-shaped: A = [1^T ; F], F iid N(0,1) (m-1) x n.
        # draw order: F, x0-raw, q, c
        F = gaussian_matrix(rng, m - 1, n)
        A = np.asfortranarray(np.vstack([np.ones((1, n)), F]))
        del F
        x0 = rng.uniform(0.5, 1.5, n) / n
        x0 /= x0.sum()                                           # exactly feasible budget row (A20)
        b = A @ x0
        b[0] = 1.0
        q = rng.uniform(0.01, 0.1, n)
        c = -rng.normal(0.05, 0.02, n)                           # 0.02 is the std (A21)
        return QPInstance(name, idx, A, q, b, c, ell, x0, None, None)

    if idx == 2:
        # SVM-shaped (A23): labels, X with rows x_i = 0.5 y_i 1_d + g_i; Xt = diag(y) X.
        # Variables [w+, w-, xi, s] (n_var = 2d + 2N); A = [Xt, -Xt, I, -I]; m = N.
        N, d = m, n
        yl = np.where(rng.uniform(size=N) < 0.5, -1.0, 1.0)
        X = gaussian_matrix(rng, N, d)
        X += 0.5 * yl[:, None]
        Xt = np.asfortranarray(yl[:, None] * X)
        del X
        nv = 2 * d + 2 * N
        q = np.concatenate([np.ones(2 * d), np.zeros(2 * N)])
        Cpen = 1.0
        c = np.concatenate([np.zeros(2 * d), Cpen * np.ones(N), np.zeros(N)])
        b = np.ones(N)
        inst = QPInstance(name, idx, None, q, b, c, ell, extra={"Xt": Xt, "labels": yl, "d": d, "N": N})
        assert inst.n == nv
        return inst

    raise ValueError(f"unknown config {idx}")


def make_general(m: int, n: int, frac_free: float = 0.2, frac_box: float = 0.3, ell: int = 20,
                 seed: int = 10) -> QPInstance:
    """Problem (P~)/(D~) with mixed variable types, SURVEY §8(f) f1 (the paper gives no
    workload; config 0's recipe extended).  vtype: 0 = I, 1 = F, 2 = J; A_ij ~ N(0, 1/n); q ~ U(0, 1);
    strictly feasible primal x0 (I: U(0.5,1.5), F: N(0,1), J: u U(0.2,0.8) with u ~ U(1,3)) and dual
    (y0 ~ N(0,1), z0_IJ ~ U(0.5,1.5), s0_J ~ U(0.5,1.5)), b = A x0, c = A^T y0 + z0 - s0 - q x0.
    Draw order: A, vtype-permutation, q, u, x0 parts, y0, z0, s0.  extra = {"vtype", "ub"}."""
    rng = np.random.default_rng(seed)
    A = gaussian_matrix(rng, m, n, 1.0 / np.sqrt(n))
    nf, nb = int(round(frac_free * n)), int(round(frac_box * n))
    perm = rng.permutation(n)
    vtype = np.zeros(n, dtype=np.int8)
    vtype[perm[:nf]] = 1
    vtype[perm[nf:nf + nb]] = 2
    F, J = vtype == 1, vtype == 2
    q = rng.uniform(0.0, 1.0, n)
    ub = np.where(J, rng.uniform(1.0, 3.0, n), 0.0)
    x0 = rng.uniform(0.5, 1.5, n)
    x0[F] = rng.standard_normal(int(F.sum()))
    x0[J] = ub[J] * rng.uniform(0.2, 0.8, int(J.sum()))
    y0 = rng.standard_normal(m)
    z0 = np.where(F, 0.0, rng.uniform(0.5, 1.5, n))
    s0 = np.where(J, rng.uniform(0.5, 1.5, n), 0.0)
    b = A @ x0
    c = A.T @ y0 + z0 - s0 - q * x0
    return QPInstance(f"gen_m{m}_n{n}_f{nf}_j{nb}", -1, A, q, b, c, ell, x0, y0, z0,
                      extra={"vtype": vtype, "ub": ub, "s0": s0})


def make_svm_dual(n_samples: int, d: int, tau: float = 1.0, ell: int = 20, seed: int = 20) -> QPInstance:
    """The paper's own SVM formulation (App. C.2): dual linear SVM
        min 1/2 v^T v - 1^T p   s.t.  v - X diag(y) p = 0,  y^T p = 0,  v free,  0 <= p <= tau,
    X (d x n_samples) a two-class Gaussian mixture, column i = (0.5 y_i 1_d + g_i) / sqrt(d) (the
    stand-in for the paper's datasets, Table 4; no dataset item is reproduced).  Variables are
    ordered [p; v] (structure 2: the dense block first): A = [-X diag(y), I_d; y^T, 0] (m = d + 1),
    dense block B = [-X diag(y); y^T], one unit block (row0 = 0, count = d, scale = +1).
    q = [0; 1_d]; c = [-1_n; 0] (reading G4: the paper prints c = [0; 1], which contradicts its
    objective -sum p_i); b = 0; vtype = [2 (J, u = tau); 1 (F)].
    Draw order: labels, G.  extra = {B, unit_blocks, vtype, ub, labels}."""
    rng = np.random.default_rng(seed)
    yl = np.where(rng.uniform(size=n_samples) < 0.5, -1.0, 1.0)
    X = gaussian_matrix(rng, d, n_samples)
    X += 0.5 * yl[None, :]
    X /= np.sqrt(d)
    B = np.asfortranarray(np.vstack([-X * yl[None, :], yl[None, :]]))
    m = d + 1
    n = n_samples + d
    q = np.concatenate([np.zeros(n_samples), np.ones(d)])
    c = np.concatenate([-np.ones(n_samples), np.zeros(d)])
    b = np.zeros(m)
    vtype = np.concatenate([np.full(n_samples, 2, np.int8), np.full(d, 1, np.int8)])
    ub = np.concatenate([np.full(n_samples, float(tau)), np.zeros(d)])
    return QPInstance(f"svmdual_n{n_samples}_d{d}", -2, None, q, b, c, ell,
                      extra={"B": B, "unit_blocks": [(0, d, 1.0)], "vtype": vtype, "ub": ub, "labels": yl})


def make_portfolio(n_assets: int, d: int, s: int, ell: int = 20, gamma: float = 1.0, seed: int = 30) -> QPInstance:
    """The paper's portfolio formulation (Sec. 5.1, App. C.1) with a factor
    model Sigma = F F^T + D:
        min -gamma^{-1} r^T x + x^T D x + y^T y  s.t.  y = F^T x,  M x <= u,  1^T x = 1,  x >= 0,  y free.
    Slacks t = u - M x >= 0 make it (P~): variables [x (n, I); y (s, F); t (d, I)], rows
    [y - F^T x = 0 (s); M x + t = u (d); 1^T x = 1 (1)], so m = s + d + 1 (50101 at the paper's
    n = 80000, d = 50000, s = 100).  Structure 2: dense block B = [-F^T; M; 1^T] (the x columns),
    unit blocks (0, s, +1) for y and (s, d, +1) for t.  q = [2 diag(D); 2 1_s; 0_d], c = [-r/gamma; 0; 0].
    Synthetic stand-in: F = V diag(sqrt(sigma)) with V an orthonormalised Gaussian
    n x s and sigma_i = 10^{-3 (i-1)/s} (rapid decay); diag(D) = 1e-3 U(0.5, 1.5) (the slow tail);
    M ~ N(0, 1); r ~ N(0, 1); u ~ U(0.1, 1) (x = 1/n is strictly feasible w.h.p.).
    Draw order: V, D, M, r, u.  extra = {B, unit_blocks, vtype, ub}."""
    rng = np.random.default_rng(seed)
    V, _ = np.linalg.qr(rng.standard_normal((n_assets, s)))
    sigma = 10.0 ** (-3.0 * np.arange(s) / max(s, 1))
    F = V * np.sqrt(sigma)[None, :]
    Dd = 1e-3 * rng.uniform(0.5, 1.5, n_assets)
    M = gaussian_matrix(rng, d, n_assets)
    r = rng.standard_normal(n_assets)
    u = rng.uniform(0.1, 1.0, d)
    B = np.asfortranarray(np.vstack([-F.T, M, np.ones((1, n_assets))]))
    m = s + d + 1
    q = np.concatenate([2.0 * Dd, 2.0 * np.ones(s), np.zeros(d)])
    c = np.concatenate([-r / gamma, np.zeros(s), np.zeros(d)])
    b = np.concatenate([np.zeros(s), u, [1.0]])
    vtype = np.concatenate([np.zeros(n_assets, np.int8), np.ones(s, np.int8), np.zeros(d, np.int8)])
    return QPInstance(f"portfolio_n{n_assets}_d{d}_s{s}", -3, None, q, b, c, ell,
                      extra={"B": B, "unit_blocks": [(0, s, 1.0), (s, d, 1.0)], "vtype": vtype,
                             "ub": np.zeros(n_assets + s + d)})


def structured_dense_A(B: np.ndarray, unit_blocks, m: int) -> np.ndarray:
    """Materialise A = [B, S_0, S_1, ...] (structure 2) for SMALL instances only (tests)."""
    cols = [np.asarray(B)]
    for row0, count, scale in unit_blocks:
        S = np.zeros((m, count))
        S[row0 + np.arange(count), np.arange(count)] = scale
        cols.append(S)
    return np.asfortranarray(np.hstack(cols))


def svm_dense_A(inst: QPInstance) -> np.ndarray:
    """Materialise A = [Xt, -Xt, I, -I] for SMALL SVM instances only (tests)."""
    Xt = inst.extra["Xt"]
    N = Xt.shape[0]
    I = np.eye(N)
    return np.asfortranarray(np.hstack([Xt, -Xt, I, -I]))
