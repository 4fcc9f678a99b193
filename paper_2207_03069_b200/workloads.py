"""Seeded synthetic QUBO instances shaped like the paper's workloads.

This module is the ONE piece shared by the oracle side (tests) and the CUDA
side (bench, tests): it only draws inputs.  It holds none of the search
method's arithmetic.  The reductions below (MaxCut, one-hot TSP/QAP) are the
*input definitions* of the paper's problems (Sec. II); tests pin
them exhaustively (E = -cut, E = C - mp) against plain definitions.

Every instance is an upper-triangular int16 matrix ``U`` (row-major n x n,
zeros below the diagonal): ``E(X) = sum_{i<=j} U_ij x_i x_j`` (Eq.(2), P:107,
reading R-1 in DESIGN.md).  Seeds feed numpy's PCG64.
"""
from __future__ import annotations

import numpy as np


def _rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(np.random.PCG64(seed))


def random_dense(n: int, seed: int, lo: int = -32767, hi: int = 32767) -> np.ndarray:
    """Random dense int16 QUBO: U_ij ~ U{lo..hi} for i <= j (configs K16, R32K).

    Row blocks keep peak host memory at ~1x the matrix for n = 32768 (2 GiB).
    """
    rng = _rng(seed)
    U = np.empty((n, n), np.int16)
    blk = max(1, min(n, (1 << 26) // max(n, 1)))
    for r0 in range(0, n, blk):
        r1 = min(n, r0 + blk)
        U[r0:r1] = rng.integers(lo, hi + 1, size=(r1 - r0, n), dtype=np.int16)
        # zero strictly-lower part of these rows
        for r in range(r0, r1):
            U[r, :r] = 0
    return U


def maxcut_qubo(n: int, edges: np.ndarray, w: np.ndarray) -> np.ndarray:
    """MaxCut -> QUBO: each edge adds w(2 x_i x_j - x_i^2 - x_j^2),
    i.e. +2w to U_ij (i<j) and -w to U_ii and U_jj, so E(X) = -cut(X)."""
    U = np.zeros((n, n), np.int64)
    i = np.minimum(edges[:, 0], edges[:, 1])
    j = np.maximum(edges[:, 0], edges[:, 1])
    np.add.at(U, (i, j), 2 * w)
    np.add.at(U, (i, i), -w)
    np.add.at(U, (j, j), -w)
    assert np.abs(U).max() <= 32767
    return U.astype(np.int16)


def gset_like(n: int = 800, m: int = 19176, seed: int = 1):
    """G-set-shaped sparse MaxCut (GS800): m distinct uniform random edges,
    weights +-1 equiprobable (config 2).  Returns (U, edges, w)."""
    rng = _rng(seed)
    seen = set()
    edges = []
    while len(edges) < m:
        a, b = rng.integers(0, n, size=2)
        if a == b:
            continue
        key = (min(a, b), max(a, b))
        if key in seen:
            continue
        seen.add(key)
        edges.append(key)
    edges = np.array(edges, np.int64)
    w = rng.choice(np.array([-1, 1], np.int64), size=m)
    return maxcut_qubo(n, edges, w), edges, w


def complete_pm1(n: int = 2000, seed: int = 1):
    """K2000-shaped complete graph with random +-1 weights (config 4)."""
    rng = _rng(seed)
    iu, ju = np.triu_indices(n, 1)
    w = rng.choice(np.array([-1, 1], np.int64), size=iu.size)
    edges = np.stack([iu, ju], 1).astype(np.int64)
    return maxcut_qubo(n, edges, w), edges, w


def qap_qubo(flow: np.ndarray, dist: np.ndarray, p: int) -> np.ndarray:
    """One-hot QAP -> QUBO in the upper-triangle convention
    (reading R-21): for bits a=<i,j> < b=<i',j'> the coefficient is
    l(i,i')d(j,j') + l(i',i)d(j',j) if i != i' and j != j'; 2p if exactly one
    of i=i', j=j' holds; the diagonal is -p.  Then E(X) = C(g_X) - m p for
    every feasible X."""
    m = flow.shape[0]
    N = m * m
    U = np.zeros((N, N), np.int64)
    for a in range(N):
        i, j = divmod(a, m)
        U[a, a] = -p
        for b in range(a + 1, N):
            i2, j2 = divmod(b, m)
            if i != i2 and j != j2:
                U[a, b] = flow[i, i2] * dist[j, j2] + flow[i2, i] * dist[j2, j]
            elif (i == i2) != (j == j2):
                U[a, b] = 2 * p
    assert np.abs(U).max() <= 32767, "QAP weights overflow int16"
    return U.astype(np.int16)


def circular_flow(m: int) -> np.ndarray:
    """TSP as QAP with a circular flow: facility i talks to i+-1."""
    f = np.zeros((m, m), np.int64)
    for i in range(m):
        f[i, (i + 1) % m] = 1
        f[(i + 1) % m, i] = 1
    return f


def cycle_metric(m: int, scale: int, seed: int) -> np.ndarray:
    """d(j,j') = scale * cyclic distance between randomly permuted labels."""
    rng = _rng(seed)
    lab = rng.permutation(m)
    a = lab[:, None]
    b = lab[None, :]
    d = np.abs(a - b)
    return (scale * np.minimum(d, m - d)).astype(np.int64)


def tsp_onehot(m: int = 32, scale: int = 10, seed: int = 1):
    """TSP32: one-hot TSP over a cycle metric (n = m^2 bits), penalty
    p = 4 max d + 1 (reading R-22).  Known optimum: tour = m*scale, and with
    the symmetric circular flow C* = 2 m scale, so E* = 2 m scale - m p.
    Returns (U, dist, p, E_star)."""
    d = cycle_metric(m, scale, seed)
    p = 4 * int(d.max()) + 1
    U = qap_qubo(circular_flow(m), d, p)
    return U, d, p, 2 * m * scale - m * p


def euclid_tsp(m: int = 32, seed: int = 1):
    """TSP over m uniform cities in [0,1000]^2, rounded Euclidean distances."""
    rng = _rng(seed)
    pts = rng.uniform(0, 1000, size=(m, 2))
    d = np.rint(np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))).astype(np.int64)
    p = 4 * int(d.max()) + 1
    return qap_qubo(circular_flow(m), d, p), d, p


def ising_to_qubo(n: int, J_edges: np.ndarray, J: np.ndarray, h: np.ndarray):
    """Ising -> QUBO with s = 2x - 1 (constructive form SPEC S:69):
    U_ij = 4 J_ij (i < j), U_ii = 2 h_i - 2 sum_j J_ij, offset = sum J - sum h, so
    E(X) + offset = H(S) for every spin vector (Eq.(1)).  Returns (U, offset)."""
    U = np.zeros((n, n), np.int64)
    i = np.minimum(J_edges[:, 0], J_edges[:, 1])
    j = np.maximum(J_edges[:, 0], J_edges[:, 1])
    np.add.at(U, (i, j), 4 * J)
    d = 2 * h.astype(np.int64)
    np.add.at(d, i, -2 * J)
    np.add.at(d, j, -2 * J)
    U[np.arange(n), np.arange(n)] += d
    assert np.abs(U).max() <= 32767
    return U.astype(np.int16), int(J.sum() - h.sum())


def qasp_like(n: int = 5627, m: int = 40279, r: int = 1, seed: int = 1):
    """QASP-shaped sparse Ising: a synthetic stand-in for
    the D-Wave Advantage 4.1 working graph (5627 nodes, 40279 edges; the real
    faulty-qubit graph is not available): local random edges (each node links to
    nodes within a window of +-64 positions, like Pegasus' bounded degree ~14),
    J uniform over the 2r nonzero integers of [-r, r], h over the 8r nonzero
    integers of [-4r, 4r].  Returns (U, offset, edges, J, h)."""
    rng = _rng(seed)
    seen = set()
    edges = []
    while len(edges) < m:
        a = int(rng.integers(0, n))
        b = int((a + rng.integers(1, 65)) % n)
        key = (min(a, b), max(a, b))
        if key in seen:
            continue
        seen.add(key)
        edges.append(key)
    edges = np.array(edges, np.int64)
    Jv = np.concatenate([np.arange(-r, 0), np.arange(1, r + 1)])
    hv = np.concatenate([np.arange(-4 * r, 0), np.arange(1, 4 * r + 1)])
    J = rng.choice(Jv, size=m)
    h = rng.choice(hv, size=n)
    U, off = ising_to_qubo(n, edges, J, h)
    return U, off, edges, J, h


def random_target(n: int, seed: int) -> np.ndarray:
    return _rng(seed).integers(0, 2, size=n, dtype=np.uint8)


# the five configs of BASELINE.json (SURVEY 8(d) recipes)
def make(config: str, seed: int = 1):
    """Return (U, meta) for a named config."""
    if config == "K16":
        return random_dense(16, seed), dict(s_milli=100, b_milli=10000, pools=1, slots=1)
    if config == "GS800":
        U, _, _ = gset_like(800, 19176, seed)
        return U, dict(s_milli=100, b_milli=10000)
    if config == "TSP32":
        U, _, _, E_star = tsp_onehot(32, 10, seed)
        return U, dict(s_milli=100, b_milli=1000, target=E_star)
    if config == "K2000s":
        U, _, _ = complete_pm1(2000, seed)
        return U, dict(s_milli=100, b_milli=10000)
    if config == "R32K":
        return random_dense(32768, seed), dict(s_milli=100, b_milli=1000)
    if config == "R64K":
        # the largest n the boundary accepts (cluster tier);
        # |U| <= 32767 keeps max_k sum_j |W_kj| <= 65536 * 32767 < 2^31 - 1
        return random_dense(65536, seed), dict(s_milli=100, b_milli=1000)
    if config.startswith("QASP"):               # QASP1 / QASP16 / QASP256 (resolution r)
        r = int(config[4:] or 1)
        U, off, _, _, _ = qasp_like(5627, 40279, r, seed)
        return U, dict(s_milli=100, b_milli=1000, offset=off, sparse=True)
    raise KeyError(config)
