"""Seeded synthetic input generators for the five BASELINE configs (C1-C5).

This module is shared by the tests, ``bench.py`` and ``smoke()``; it holds NONE of the
method's arithmetic (no local solve, no sweeps, no marching) -- only the speed field F,
the exit mask and the exit values q that define an instance of Eq. (1)
("|grad u| F = 1 on Omega, u = q on Q") on the grid of P:95-100
(x_ijk = (ih, jh, kh), 0 <= i,j,k <= n, nh = 1, M = (n+1)^3).

Layout (ABI): arrays of shape (n+1, n+1, n+1) indexed
[k, j, i] in C order, so the flat index is idx = i + (n+1)*(j + (n+1)*k) (i fastest).

Recipes (readings R22-R24 in DESIGN.md):
  C1  F = 1, exit (n/2, n/2, n/2)                        -- Ex.1 shape
  C2  F = 1 + 0.5 sin(8 pi x) sin(8 pi y) sin(8 pi z), exit at centre -- Ex.2 shape
  C3  checkerboard of 8^3 blocks of side 1/8, F in {1, 10}, exit (0,0,0) -- P:1596-1599 shape
  C4  F = 1 with 8 planar F = 0 walls, 4 random square holes each, exit face k = 0
      -- shell-maze shape, made planar/impermeable (R11, R23)
  C5  F = clip(1 + sum_b a_b exp(-|x-c_b|^2 / (2 sigma_b^2)), 0.3, 2), 64 random exits (R24)
All exits have q = 0 (D.2). F is generated once in fp64; fp32 runs use F.astype(float32).
The paper uses no dataset: every workload is an analytic F, so these
generators ARE the workloads; nothing stands in for a public benchmark.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------------------
# Config table (BASELINE.json "configs"; SURVEY.md 8 per-config sizes)
# --------------------------------------------------------------------------------------
CONFIGS = {
    "C1": dict(n=128, precisions=("f64",), cell_sizes=(8,)),
    "C2": dict(n=256, precisions=("f64", "f32"), cell_sizes=(8, 16)),
    "C3": dict(n=512, precisions=("f32", "f64"), cell_sizes=(16,)),
    "C4": dict(n=512, precisions=("f32",), cell_sizes=(16,)),
    "C5": dict(n=1024, precisions=("f32", "f64"), cell_sizes=(16,)),
}

C4_SEED = 1306  # R23: numpy.random.default_rng(1306)
C5_SEED = 4743  # R24: numpy.random.default_rng(4743)


@dataclass
class Workload:
    name: str
    n: int
    F: np.ndarray           # (n+1)^3 float64, [k, j, i]
    exit_mask: np.ndarray   # (n+1)^3 uint8
    exit_vals: np.ndarray   # (n+1)^3 float64 (q; read where mask == 1)
    meta: dict = field(default_factory=dict)

    @property
    def h(self) -> float:
        return float(self.meta.get("h", 1.0 / self.n))

    @property
    def M(self) -> int:
        return (self.n + 1) ** 3

    def f_sha256(self) -> str:
        return hashlib.sha256(np.ascontiguousarray(self.F).tobytes()).hexdigest()

    def as_dtype(self, dtype):
        """(F, exit_mask, exit_vals) in the run precision (round-to-nearest cast, D.2)."""
        return (np.ascontiguousarray(self.F.astype(dtype)), self.exit_mask,
                np.ascontiguousarray(self.exit_vals.astype(dtype)))


def _axis(n: int) -> np.ndarray:
    # x_i = i*h with h = 1/n; for n a power of two i/n is exact
    return np.arange(n + 1, dtype=np.float64) / n


def _point_exits(n: int, pts) -> tuple[np.ndarray, np.ndarray]:
    mask = np.zeros((n + 1,) * 3, dtype=np.uint8)
    for (i, j, k) in pts:
        mask[k, j, i] = 1
    return mask, np.zeros((n + 1,) * 3, dtype=np.float64)


def c1(n: int = 128) -> Workload:
    """C1: F = 1, single exit at the grid centre (n even)."""
    assert n % 2 == 0
    F = np.ones((n + 1,) * 3, dtype=np.float64)
    c = n // 2
    mask, q = _point_exits(n, [(c, c, c)])
    return Workload("C1", n, F, mask, q, dict(exit=(c, c, c)))


def c2(n: int = 256) -> Workload:
    """C2: F = 1 + 0.5 sin(8 pi x) sin(8 pi y) sin(8 pi z) in [0.5, 1.5], centre exit."""
    assert n % 2 == 0
    x = _axis(n)
    s = np.sin(8.0 * np.pi * x)
    F = 1.0 + 0.5 * (s[:, None, None] * s[None, :, None] * s[None, None, :])
    c = n // 2
    mask, q = _point_exits(n, [(c, c, c)])
    return Workload("C2", n, np.ascontiguousarray(F), mask, q, dict(exit=(c, c, c)))


def c3_block_index(n: int) -> np.ndarray:
    """R22: b(i) = min(floor(i / (n/8)), 7); a block face plane belongs to the + side."""
    assert n % 8 == 0
    return np.minimum(np.arange(n + 1) // (n // 8), 7)


def c3(n: int = 512, fast: float = 10.0) -> Workload:
    """C3: 8^3 checkerboard, F = 1 where b(i)+b(j)+b(k) is even (the exit block), else `fast`."""
    b = c3_block_index(n)
    par = (b[:, None, None] + b[None, :, None] + b[None, None, :]) % 2
    F = np.where(par == 0, 1.0, fast).astype(np.float64)
    mask, q = _point_exits(n, [(0, 0, 0)])
    return Workload("C3", n, np.ascontiguousarray(F), mask, q, dict(exit=(0, 0, 0), fast=fast))


def c4_geometry(n: int = 512, seed: int = C4_SEED):
    """R23: wall planes k_m = round((m + 1/2) n / 9), m = 0..7; each wall has 4 square holes of
    n/16 x n/16 points [i0, i0+w) x [j0, j0+w), (i0, j0) = rng.integers(0, n + 2 - w, size=2),
    drawn for m = 0..7 then hole 0..3 (overlaps allowed)."""
    assert n % 16 == 0
    w = n // 16
    rng = np.random.default_rng(seed)
    walls = [int(np.floor((m + 0.5) * n / 9.0 + 0.5)) for m in range(8)]
    holes = []
    for m in range(8):
        hm = []
        for _ in range(4):
            i0, j0 = rng.integers(0, n + 2 - w, size=2)
            hm.append((int(i0), int(j0)))
        holes.append(hm)
    return walls, holes, w


def c4(n: int = 512, seed: int = C4_SEED) -> Workload:
    """C4: F = 1 except 8 one-point-thick F = 0 walls pierced by 4 holes; exits = face k = 0."""
    walls, holes, w = c4_geometry(n, seed)
    F = np.ones((n + 1,) * 3, dtype=np.float64)
    for km, hm in zip(walls, holes):
        plane = np.zeros((n + 1, n + 1), dtype=np.float64)  # [j, i]
        for (i0, j0) in hm:
            plane[j0:j0 + w, i0:i0 + w] = 1.0
        F[km] = plane
    mask = np.zeros((n + 1,) * 3, dtype=np.uint8)
    mask[0] = 1
    q = np.zeros((n + 1,) * 3, dtype=np.float64)
    return Workload("C4", n, F, mask, q, dict(walls=walls, holes=holes, hole=w, seed=seed))


def c5_params(n: int = 1024, seed: int = C5_SEED):
    """R24: rng = default_rng(4743); draw a, c, sigma, exits in that order; dedupe exits."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(-0.4, 0.4, 32)
    c = rng.uniform(0.0, 1.0, (32, 3))
    sig = rng.uniform(0.03, 0.15, 32)
    E = rng.integers(0, n + 1, (64, 3))
    seen, ex = set(), []
    for e in map(tuple, E.tolist()):
        if e not in seen:
            seen.add(e)
            ex.append(e)
    return a, c, sig, ex


def c5_field_torch(n: int, a, c, sig, device="cpu", dtype=None, slab: int = 32):
    """F of C5 evaluated in fp64 with torch (z-slabs), returned as a torch tensor [k, j, i]
    on `device` in `dtype` (default fp64). Plumbing only: the formula is the workload's."""
    import torch
    dtype = dtype or torch.float64
    x = torch.arange(n + 1, dtype=torch.float64, device=device) / n
    out = torch.empty((n + 1,) * 3, dtype=dtype, device=device)
    a_t = torch.tensor(a, dtype=torch.float64, device=device)
    c_t = torch.tensor(c, dtype=torch.float64, device=device)
    s_t = torch.tensor(sig, dtype=torch.float64, device=device)
    inv = 1.0 / (2.0 * s_t * s_t)
    dx2 = (x[None, :] - c_t[:, 0:1]) ** 2  # [32, n+1] over i
    dy2 = (x[None, :] - c_t[:, 1:2]) ** 2  # over j
    dz2 = (x[None, :] - c_t[:, 2:3]) ** 2  # over k
    for k0 in range(0, n + 1, slab):
        k1 = min(n + 1, k0 + slab)
        acc = torch.ones((k1 - k0, n + 1, n + 1), dtype=torch.float64, device=device)
        for b in range(32):
            e = (dz2[b, k0:k1, None, None] + dy2[b, None, :, None] + dx2[b, None, None, :])
            acc += a_t[b] * torch.exp(-e * inv[b])
        out[k0:k1] = acc.clamp_(0.3, 2.0).to(dtype)
    return out


def c5(n: int = 1024, seed: int = C5_SEED) -> Workload:
    """C5 on the host (fp64 numpy). For n = 1024 prefer c5_field_torch on the GPU."""
    a, c, sig, ex = c5_params(n, seed)
    F = c5_field_torch(n, a, c, sig).numpy()
    mask, q = _point_exits(n, ex)
    return Workload("C5", n, F, mask, q, dict(exits=ex, seed=seed))


GENERATORS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


def make(name: str, n: int | None = None) -> Workload:
    """Build config `name` at its BASELINE size, or at the reduced size n (same formulas)."""
    gen = GENERATORS[name]
    return gen() if n is None else gen(n)


def random_instance(n: int, seed: int, p_wall: float = 0.15, n_exits: int = 3,
                    fmin: float = 0.25, fmax: float = 4.0, q_max: float = 0.0) -> Workload:
    """Small random instances for oracle self-tests and parity: random F with F = 0 obstacles,
    random exits (some with q > 0 if q_max > 0)."""
    rng = np.random.default_rng(seed)
    shp = (n + 1,) * 3
    F = rng.uniform(fmin, fmax, shp)
    F[rng.random(shp) < p_wall] = 0.0
    mask = np.zeros(shp, dtype=np.uint8)
    q = np.zeros(shp, dtype=np.float64)
    flat = rng.choice((n + 1) ** 3, size=n_exits, replace=False)
    mask.reshape(-1)[flat] = 1
    if q_max > 0:
        q.reshape(-1)[flat] = rng.uniform(0.0, q_max, n_exits)
    return Workload(f"rand{n}_{seed}", n, F, mask, q, dict(seed=seed))


# --------------------------------------------------------------------------------------
# The paper's own workload suite: M = N^3 points per side N on the unit
# cube (h = 1/(N-1)); N even, so the exit set is the 8 gridpoints closest to the centre
# ("we have initialized U on the set Q of the 8 gridpoints closest to the center").
# --------------------------------------------------------------------------------------
def _centre8(N: int):
    assert N % 2 == 0, "the paper's centre-exit problems use an even number of points per side"
    lo, hi = N // 2 - 1, N // 2
    return [(i, j, k) for i in (lo, hi) for j in (lo, hi) for k in (lo, hi)]


def paper_example(ex: int, N: int) -> Workload:
    """Examples 1-3 of P:760-764 on N^3 points: F = 1; 1 + .5 sin(20 pi x) sin(20 pi y)
    sin(20 pi z); 1 + .99 sin(2 pi x) sin(2 pi y) sin(2 pi z); q = 0 on the 8 centre points."""
    n = N - 1
    x = np.arange(N, dtype=np.float64) / n
    if ex == 1:
        F = np.ones((N,) * 3)
    else:
        a, w = (0.5, 20.0) if ex == 2 else (0.99, 2.0)
        sv = np.sin(w * np.pi * x)
        F = 1.0 + a * (sv[:, None, None] * sv[None, :, None] * sv[None, None, :])
    mask, q = _point_exits(n, _centre8(N))
    return Workload(f"Ex{ex}_{N}", n, np.ascontiguousarray(F), mask, q, dict(ex=ex, N=N))


def paper_checkerboard(K: int, N: int) -> Workload:
    """3D checkerboard of P:1596-1600: K^3 checkers of edge 1/K, F = 2 on black and 1 on white
    checkers, centre exit (8 points).  Reading: black = checkers with odd bx+by+bz (the centre
    checker for odd K); a gridpoint on a checker boundary takes the checker floor(x K) (the
    paper picks grids avoiding this, P:1597 footnote)."""
    n = N - 1
    x = np.arange(N, dtype=np.float64) / n
    b = np.minimum(np.floor(x * K).astype(np.int64), K - 1)
    par = (b[:, None, None] + b[None, :, None] + b[None, None, :]) % 2
    F = np.where(par == 1, 2.0, 1.0)
    mask, q = _point_exits(n, _centre8(N))
    return Workload(f"CB{K}_{N}", n, np.ascontiguousarray(F), mask, q, dict(K=K, N=N))


def paper_shell_maze(N: int, t: float = 1.0 / 12, w: float = 0.1, slow: float = 0.001) -> Workload:
    """Permeable spherical-shell maze of P:1627-1636 on [-1,1]^3 (h = 2/(N-1)): F = 1 outside
    four barriers A_1..A_4 (radii .3/.5/.7/.9, thickness t, openings x^2 + y^2 < w on
    alternating sides z < 0 / z > 0) and F = .001 inside them; exits at the gridpoint(s)
    closest to the origin (8 for even N)."""
    n = N - 1
    x = -1.0 + 2.0 * np.arange(N, dtype=np.float64) / n
    X = x[None, None, :]
    Y = x[None, :, None]
    Z = x[:, None, None]
    rad = np.sqrt(X * X + Y * Y + Z * Z)
    hole = (X * X + Y * Y) < w
    F = np.ones((N,) * 3)
    for r0, neg in ((0.3, True), (0.5, False), (0.7, True), (0.9, False)):
        shell = (rad > r0) & (rad < r0 + t)
        opening = hole & ((Z < 0) if neg else (Z > 0))
        F[shell & ~opening] = slow
    if N % 2 == 0:
        ex = _centre8(N)
    else:
        ex = [(n // 2,) * 3]
    mask, q = _point_exits(n, ex)
    return Workload(f"Maze_{N}", n, np.ascontiguousarray(F), mask, q, dict(N=N, h=2.0 / n))
