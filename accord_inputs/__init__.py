"""Seeded synthetic inputs for the ACCORD-FBS hot path (shared by oracle tests,
GPU parity tests, smoke() and bench.py).

This module holds NONE of the method's arithmetic (no gradient, prox, objective
or line search). It only builds ground-truth precision matrices Omega0 and draws
data X with rows iid N(0, Omega0^{-1}), then centers the columns
("X ... is the centered data matrix").

Recipes (BASELINE.json `configs`, SURVEY.md §8(d) "Common generator"):
  * chain: tridiagonal Omega0, omega_ii = 1, omega_{i,i+-1} = rho (BJ config 1;
    PAPER.md:763-770, §5.4 chain graph).
  * BA(m=1) scale-free tree blocks: node 1 attaches to node 0, node t >= 2 to an
    earlier node j with probability deg(j)/sum(deg) (preferential attachment).
    Edge weights s*u with u ~ U[wlo, whi], s = +-1 w.p. 1/2;
    diagonal = 1.5 * row abs-sum, then D^{-1/2} Omega D^{-1/2}
    for a unit diagonal (BJ configs 2-5).
  * hubs (BJ config 4): in each block, 1% of nodes become hubs joined to ~50
    random in-block neighbours with the same weight law, before the diagonal is
    set (SURVEY.md §8(c) ambiguity row 17: hubs placed inside blocks).
  * sampling: Omega0 = U U^T with U upper triangular, x = U^{-T} z,
    z ~ N(0, I) (the triangular-factor sampler of PAPER.md:591). For tree blocks
    U has one off-diagonal per column (perfect elimination order, no fill) and
    the solve is O(b) per sample; other blocks use a dense Cholesky.

RNG: numpy PCG64 `default_rng(seed)`; graph seed = 1000 + c, sample seed =
2000 + c for BJ config c.

Data are returned VARIABLE-MAJOR: Xt is p x n row-major (Xt[j, m] = X[m, j]),
i.e. X stored column-major. `X = Xt.T` is the paper's sample-major n x p matrix.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Config", "CONFIGS", "TEST_CONFIGS", "get_config", "ba_tree_parents",
    "make_omega0", "sample_xt", "center_rows", "make_problem", "Problem",
    "xt_sha256",
]


@dataclass(frozen=True)
class Config:
    name: str
    p: int
    n: int
    dtype: str               # "f64" or "f32": dtype of X handed to the solver
    structure: str           # "chain" | "ba" | "ba_hubs"
    block: int               # block size (p for a single block)
    lambdas: tuple           # lambda values (BJ)
    T: int                   # fixed iteration count (BJ)
    graph_seed: int
    sample_seed: int
    tau0: float = 0.5        # SURVEY.md §8(c) ambiguity row 6
    beta: float = 0.5        # SURVEY.md §8(c) ambiguity row 5
    rho: float = 0.4         # chain off-diagonal
    hub_frac: float = 0.01
    hub_degree: int = 50
    extra: dict = field(default_factory=dict, compare=False, hash=False)


def _cfg(c, **kw):
    return Config(graph_seed=1000 + c, sample_seed=2000 + c, **kw)


# BASELINE.json `configs` (1-based, as in BJ).
CONFIGS = {
    1: _cfg(1, name="c1_chain_p100_n50_f64", p=100, n=50, dtype="f64",
            structure="chain", block=100, lambdas=(0.1,), T=50),
    2: _cfg(2, name="c2_ba_p2000_n500_f32", p=2000, n=500, dtype="f32",
            structure="ba", block=2000, lambdas=(0.05, 0.1, 0.2), T=100),
    3: _cfg(3, name="c3_ba20x1000_p20000_n1000_f32", p=20000, n=1000,
            dtype="f32", structure="ba", block=1000, lambdas=(0.1,), T=100),
    4: _cfg(4, name="c4_ba100x1000_hubs_p100000_n2000_f32", p=100000, n=2000,
            dtype="f32", structure="ba_hubs", block=1000, lambdas=(0.1,), T=50),
    5: _cfg(5, name="c5_ba1000x1000_p1000000_n1000_f32", p=1000000, n=1000,
            dtype="f32", structure="ba", block=1000, lambdas=(0.15,), T=20),
    # Optional "TCGA-shaped" stand-in: the shape and lambda of
    # the paper's TCGA LIHC case study (p = 285,358 probes, n = 365 samples,
    # lambda = 0.45) on synthetic block-diagonal data with
    # small local blocks (genome-ordered probes), standardized
    # columns. No TCGA values are used.
    6: _cfg(6, name="c6_tcga_shaped_p285358_n365_f32", p=285358, n=365,
            dtype="f32", structure="ba", block=500, lambdas=(0.45,), T=20,
            extra={"standardize": True}),
}

# Small cases of the same recipes, for tests that must finish in seconds.
# Shapes are chosen to span several GEMM tiles plus ragged tails (p, n not
# multiples of 128/64).
TEST_CONFIGS = {
    "t_chain": Config(name="t_chain_p37_n23_f64", p=37, n=23, dtype="f64",
                      structure="chain", block=37, lambdas=(0.1,), T=10,
                      graph_seed=11, sample_seed=12),
    "t_ba_f64": Config(name="t_ba_p300_n130_f64", p=300, n=130, dtype="f64",
                       structure="ba", block=150, lambdas=(0.1,), T=15,
                       graph_seed=21, sample_seed=22),
    "t_ba_f32": Config(name="t_ba_p700_n250_f32", p=700, n=250, dtype="f32",
                       structure="ba", block=350, lambdas=(0.1,), T=20,
                       graph_seed=31, sample_seed=32),
    "t_hubs_f32": Config(name="t_hubs_p1100_n333_f32", p=1100, n=333,
                         dtype="f32", structure="ba_hubs", block=550,
                         lambdas=(0.1,), T=10, graph_seed=41, sample_seed=42,
                         hub_degree=20),
    "t_mid_f32": Config(name="t_mid_p3000_n1000_f32", p=3000, n=1000,
                        dtype="f32", structure="ba", block=1000,
                        lambdas=(0.1,), T=10, graph_seed=51, sample_seed=52),
}


def get_config(key) -> Config:
    if isinstance(key, int) or (isinstance(key, str) and key.isdigit()):
        return CONFIGS[int(key)]
    if key in TEST_CONFIGS:
        return TEST_CONFIGS[key]
    for c in list(CONFIGS.values()) + list(TEST_CONFIGS.values()):
        if c.name == key:
            return c
    raise KeyError(key)


# ----------------------------------------------------------------------------
# Graph structure
# ----------------------------------------------------------------------------

def ba_tree_parents(b: int, rng: np.random.Generator) -> np.ndarray:
    """Barabasi-Albert (m=1) tree on b nodes; returns parent[t] (< t) for
    t >= 1 and parent[0] = -1. Node t attaches to j < t with probability
    deg(j) / sum(deg) (preferential attachment)."""
    parent = np.full(b, -1, dtype=np.int64)
    if b <= 1:
        return parent
    # Sampling proportional to degree == picking a uniform endpoint of a
    # uniformly chosen existing edge-end ("repeated nodes" list).
    ends = np.empty(2 * (b - 1), dtype=np.int64)
    parent[1] = 0
    ends[0], ends[1] = 0, 1
    m = 2
    u = rng.random(b)
    for t in range(2, b):
        j = ends[int(u[t] * m)]
        parent[t] = j
        ends[m], ends[m + 1] = j, t
        m += 2
    return parent


def _weights(rng, k, wlo, whi):
    s = np.where(rng.random(k) < 0.5, -1.0, 1.0)
    return s * rng.uniform(wlo, whi, size=k)


@dataclass
class Block:
    """One diagonal block of Omega0 (local indices 0..b-1)."""
    b: int
    rows: np.ndarray     # COO of the symmetric off-diagonal part (both triangles)
    cols: np.ndarray
    vals: np.ndarray
    diag: np.ndarray
    parent: np.ndarray | None   # set iff the block graph is a tree with parent < child

    def dense(self) -> np.ndarray:
        A = np.zeros((self.b, self.b))
        A[self.rows, self.cols] = self.vals
        A[np.arange(self.b), np.arange(self.b)] = self.diag
        return A


def _unit_diag(b, r, c, w, dom=1.5):
    """diagonal = dom * row abs-sum, then unit-diagonal
    rescaling D^{-1/2} Omega D^{-1/2}."""
    absrow = np.zeros(b)
    np.add.at(absrow, r, np.abs(w))
    d = dom * absrow
    d[d == 0] = 1.0          # isolated node (b == 1)
    s = 1.0 / np.sqrt(d)
    return w * s[r] * s[c], np.ones(b)


def _ba_block(b, rng, wlo, whi, hubs=0, hub_degree=50):
    parent = ba_tree_parents(b, rng)
    child = np.arange(1, b)
    par = parent[1:]
    w = _weights(rng, b - 1, wlo, whi)
    edges = {(int(min(x, y)), int(max(x, y))): float(v)
             for x, y, v in zip(child, par, w)}
    tree = hubs == 0
    if hubs > 0:
        hub_nodes = rng.choice(b, size=hubs, replace=False)
        for h in hub_nodes:
            cand = rng.permutation(b)
            added = 0
            for j in cand:
                if added >= hub_degree:
                    break
                j = int(j)
                if j == h:
                    continue
                key = (min(h, j), max(h, j))
                if key in edges:
                    continue
                edges[key] = float(_weights(rng, 1, wlo, whi)[0])
                added += 1
    keys = np.array(sorted(edges.keys()), dtype=np.int64).reshape(-1, 2)
    vals = np.array([edges[tuple(k)] for k in keys])
    r = np.concatenate([keys[:, 0], keys[:, 1]])
    c = np.concatenate([keys[:, 1], keys[:, 0]])
    w = np.concatenate([vals, vals])
    w, diag = _unit_diag(b, r, c, w)
    return Block(b, r, c, w, diag, parent if tree else None)


def _chain_block(b, rho):
    i = np.arange(b - 1)
    r = np.concatenate([i, i + 1])
    c = np.concatenate([i + 1, i])
    w = np.full(2 * (b - 1), rho)
    parent = np.arange(-1, b - 1)
    return Block(b, r, c, w, np.ones(b), parent)


def make_omega0(cfg: Config, wlo=0.3, whi=0.6):
    """List of diagonal blocks of the ground-truth Omega0 (block-diagonal)."""
    rng = np.random.default_rng(cfg.graph_seed)
    # equal blocks; a smaller last block when the block size does not divide p
    nb = -(-cfg.p // cfg.block)
    sizes = [cfg.block] * (nb - 1) + [cfg.p - (nb - 1) * cfg.block]
    blocks = []
    for b in sizes:
        if cfg.structure == "chain":
            blocks.append(_chain_block(b, cfg.rho))
        elif cfg.structure == "ba":
            blocks.append(_ba_block(b, rng, wlo, whi))
        elif cfg.structure == "ba_hubs":
            nh = max(1, int(round(cfg.hub_frac * b)))
            blocks.append(_ba_block(b, rng, wlo, whi, nh, min(cfg.hub_degree, b - 1)))
        else:
            raise ValueError(cfg.structure)
    return blocks


def omega0_dense(blocks) -> np.ndarray:
    p = sum(b.b for b in blocks)
    A = np.zeros((p, p))
    o = 0
    for b in blocks:
        A[o:o + b.b, o:o + b.b] = b.dense()
        o += b.b
    return A


# ----------------------------------------------------------------------------
# Sampling x ~ N(0, Omega0^{-1}) by a triangular factor
# ----------------------------------------------------------------------------

def _tree_factor(blk: Block):
    """Omega = U U^T, U upper triangular with U[t,t] = ud[t] and
    U[parent(t), t] = uo[t] (no fill for a tree with parent < child)."""
    b = blk.b
    par = blk.parent
    off = {}
    for r, c, v in zip(blk.rows, blk.cols, blk.vals):
        off[(int(r), int(c))] = float(v)
    ud = np.zeros(b)
    uo = np.zeros(b)
    acc = blk.diag.astype(np.float64).copy()   # Omega_tt - sum_children U[t,c]^2
    for t in range(b - 1, -1, -1):
        ud[t] = np.sqrt(acc[t])
        if par[t] >= 0:
            uo[t] = off[(int(par[t]), t)] / ud[t]
            acc[par[t]] -= uo[t] ** 2
    return ud, uo


def sample_xt(cfg: Config, blocks, chunk_blocks: int = 64) -> np.ndarray:
    """Draw Xt (p x n, float64, uncentered) with columns of X = Xt.T iid
    N(0, Omega0^{-1}). Solves U^T x = z per sample."""
    rng = np.random.default_rng(cfg.sample_seed)
    p, n = cfg.p, cfg.n
    Xt = np.empty((p, n), dtype=np.float64)
    o = 0
    i = 0
    while i < len(blocks):
        grp = blocks[i:i + chunk_blocks]
        b = grp[0].b
        same_tree = all(g.parent is not None and g.b == b for g in grp)
        if same_tree:
            nbk = len(grp)
            Z = rng.standard_normal((nbk, b, n))
            facs = [_tree_factor(g) for g in grp]
            ud = np.stack([f[0] for f in facs])          # nbk x b
            uo = np.stack([f[1] for f in facs])
            par = np.stack([g.parent for g in grp])
            out = np.empty((nbk, b, n))
            ar = np.arange(nbk)
            out[:, 0, :] = Z[:, 0, :] / ud[:, 0:1]
            for t in range(1, b):
                xp = out[ar, par[:, t], :]
                out[:, t, :] = (Z[:, t, :] - uo[:, t:t + 1] * xp) / ud[:, t:t + 1]
            Xt[o:o + nbk * b] = out.reshape(nbk * b, n)
            o += nbk * b
            i += nbk
        else:
            import scipy.linalg as sla
            g = grp[0]
            Z = rng.standard_normal((g.b, n))
            A = g.dense()
            # Omega = L L^T (lower); x = L^{-T} z has covariance (L L^T)^{-1}.
            L = np.linalg.cholesky(A)
            Xt[o:o + g.b] = sla.solve_triangular(L, Z, trans="T", lower=True)
            o += g.b
            i += 1
    return Xt


def center_rows(Xt: np.ndarray) -> np.ndarray:
    """Center each variable (row of Xt == column of X) in float64
    (SURVEY.md §8(c) ambiguity row 12)."""
    return Xt - Xt.mean(axis=1, keepdims=True)


@dataclass
class Problem:
    cfg: Config
    Xt: np.ndarray           # p x n, cfg dtype, centered, C-contiguous
    blocks: list

    @property
    def X(self):             # sample-major n x p view (the paper's X)
        return self.Xt.T


def make_problem(cfg, with_blocks: bool = True) -> Problem:
    cfg = get_config(cfg) if not isinstance(cfg, Config) else cfg
    blocks = make_omega0(cfg)
    Xt = center_rows(sample_xt(cfg, blocks))
    if cfg.extra.get("standardize"):   # unit-variance variables (c6)
        Xt /= np.sqrt((Xt * Xt).mean(axis=1, keepdims=True))
    dt = np.float64 if cfg.dtype == "f64" else np.float32
    Xt = np.ascontiguousarray(Xt.astype(dt))
    return Problem(cfg, Xt, blocks if with_blocks else [])


def xt_sha256(Xt: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(Xt).tobytes()).hexdigest()
