"""Seeded synthetic inputs for the coarse-grid Dirac operator (DESIGN.md §3 "Input recipe").

This module is the ONE input generator shared by ``tests/``, ``oracle/`` callers and
``bench.py``.  It holds none of the operator's arithmetic: only a counter-based hash
(splitmix64) of GLOBAL indices and the recipes that turn hash values into link
matrices and colour-spinor vectors.  The CUDA library has its own, independently
written device generator (``coarse_links_generate`` / ``coarse_field_generate``); a
GPU test checks the two bit-for-bit on sampled elements.

Generator::

    splitmix64(z): z += 0x9E3779B97F4A7C15; z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                   z = (z ^ (z >> 27)) * 0x94D049BB133111EB; return z ^ (z >> 31)   (mod 2^64)
    base(seed, tag) = splitmix64(seed ^ (tag << 56))
    u(seed, tag, ctr) = ((int64)(splitmix64(base + ctr) >> 42) - 2^21) * 2^-21     in [-1, 1)

``u`` lies on a 2^-21 grid, so every value (and the tau3-hermitian symmetrisation
``(G + tau3 G^H tau3)/2`` on a 2^-22 grid) is exactly representable in fp32: fp32 storage
introduces no input rounding.

Counters (``gsite`` = global lexicographic site index, x0 fastest, Listing 2;
``part`` 0 = re, 1 = im):
    vectors: ((gsite * N + i) * 2 + part)
    links:   ((((gsite * 9 + k) * N + i) * N + j) * 2 + part)
Hop index k = 2*mu + dir (dir 0 = +mu, dir 1 = -mu), k = 8 is the diagonal X
(§6.3 "mu*2+dir"; reading R3/R8).

Tags: 1 = links, 2 = v, 3 = w, 4 = translation-invariant links.
Seeds: links 0x1612, vectors 0x7873.
"""
from __future__ import annotations

import numpy as np

SEED_LINKS = 0x1612
SEED_VEC = 0x7873
TAG_LINKS, TAG_V, TAG_W, TAG_TI = 1, 2, 3, 4

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

LINK_KINDS = ("general", "hermitian", "ti_general", "ti_hermitian")


def splitmix64(z):
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def base(seed: int, tag: int) -> np.uint64:
    return splitmix64(np.uint64((seed ^ (tag << 56)) & 0xFFFFFFFFFFFFFFFF))


def uniform(seed: int, tag: int, ctr) -> np.ndarray:
    """u(seed, tag, ctr) in [-1, 1) on a 2^-21 grid, float64 (exact in fp32)."""
    b = base(seed, tag)
    with np.errstate(over="ignore"):
        h = splitmix64(b + np.asarray(ctr, dtype=np.uint64))
    q = (h >> np.uint64(42)).astype(np.int64) - (1 << 21)
    return q.astype(np.float64) * (2.0 ** -21)


def volume(dims) -> int:
    d = [int(x) for x in dims]
    return d[0] * d[1] * d[2] * d[3]


def site_index(dims, x) -> np.ndarray:
    """Global lexicographic index, x0 fastest (Listing 2)."""
    L0, L1, L2, _ = (int(v) for v in dims)
    x = np.asarray(x, dtype=np.int64)
    return ((x[..., 3] * L2 + x[..., 2]) * L1 + x[..., 1]) * L0 + x[..., 0]


def site_coords(dims, s) -> np.ndarray:
    L0, L1, L2, _ = (int(v) for v in dims)
    s = np.asarray(s, dtype=np.int64)
    x0 = s % L0
    t = s // L0
    x1 = t % L1
    t = t // L1
    x2 = t % L2
    x3 = t // L2
    return np.stack([x0, x1, x2, x3], axis=-1)


def _sites(dims, sites):
    if sites is None:
        return np.arange(volume(dims), dtype=np.int64)
    return np.asarray(sites, dtype=np.int64).reshape(-1)


def vector(dims, N: int, seed: int = SEED_VEC, tag: int = TAG_V, sites=None) -> np.ndarray:
    """Colour-spinor field v[gsite][i], complex128, values on the 2^-21 grid.

    ``sites`` selects global site indices (default: all, in lexicographic order)."""
    g = _sites(dims, sites)
    i = np.arange(N, dtype=np.int64)
    ctr = ((g[:, None] * N + i[None, :]) * 2)[..., None] + np.arange(2, dtype=np.int64)
    u = uniform(seed, tag, ctr.astype(np.uint64))
    return u[..., 0] + 1j * u[..., 1]


def _raw_G(gsites, ks, N, seed, tag):
    """G(gsite, k)[i][j] as complex128 array [len(gsites), len(ks), N, N]."""
    g = np.asarray(gsites, dtype=np.int64)
    k = np.asarray(ks, dtype=np.int64)
    i = np.arange(N, dtype=np.int64)
    ctr = ((((g[:, None, None, None] * 9 + k[None, :, None, None]) * N + i[None, None, :, None]) * N
            + i[None, None, None, :]) * 2)
    ctr = ctr[..., None] + np.arange(2, dtype=np.int64)
    u = uniform(seed, tag, ctr.astype(np.uint64))
    return u[..., 0] + 1j * u[..., 1]


def tau3_signs(N: int) -> np.ndarray:
    """sigma(i) = +1 for i < Nvec (coarse spin 0), -1 otherwise (Listing 3: spin slower)."""
    nvec = N // 2
    return np.where(np.arange(N) < nvec, 1.0, -1.0)


def links(dims, N: int, seed: int = SEED_LINKS, kind: str = "general", scale_log2: int = 0,
          sites=None) -> np.ndarray:
    """Link field L[gsite][k][i][j] (complex128), canonical layout, for the chosen recipe.

    kind:
      general      L_k(x) = G(x, k)
      hermitian    L_{2mu}(x) = G(x, 2mu); L_{2mu+1}(x) = tau3 G(x - mu, 2mu)^H tau3;
                   X(x) = (G(x,8) + tau3 G(x,8)^H tau3) / 2     (tau3-hermitian, R5)
      ti_general / ti_hermitian   the same with gsite := 0 and tag 4 (translation invariant)
    scale_log2: multiply every entry by 2^scale_log2 (exact).
    """
    if kind not in LINK_KINDS:
        raise ValueError(kind)
    g = _sites(dims, sites)
    ti = kind.startswith("ti_")
    tag = TAG_TI if ti else TAG_LINKS
    herm = kind.endswith("hermitian")
    n = len(g)
    if ti:
        G = np.broadcast_to(_raw_G([0], range(9), N, seed, tag), (n, 9, N, N)).copy()
    else:
        G = _raw_G(g, range(9), N, seed, tag)
    if herm:
        sig = tau3_signs(N)
        ss = sig[:, None] * sig[None, :]
        out = np.empty_like(G)
        out[:, 8] = 0.5 * (G[:, 8] + ss * np.conj(np.swapaxes(G[:, 8], -1, -2)))
        x = site_coords(dims, g)
        for mu in range(4):
            out[:, 2 * mu] = G[:, 2 * mu]
            if ti:
                Gb = G[:, 2 * mu]
            else:
                xb = x.copy()
                xb[:, mu] = (xb[:, mu] - 1) % int(dims[mu])
                Gb = _raw_G(site_index(dims, xb), [2 * mu], N, seed, tag)[:, 0]
            out[:, 2 * mu + 1] = ss * np.conj(np.swapaxes(Gb, -1, -2))
        G = out
    if scale_log2:
        G = G * (2.0 ** scale_log2)
    return G
