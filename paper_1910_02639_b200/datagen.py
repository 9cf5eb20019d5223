"""Seeded synthetic particle sets for the five BASELINE.json configurations.

This module holds NO arithmetic of the method (no tree, no cell keys, no
distance test): it only draws positions and smoothing lengths.  It is the one
module shared by the CUDA path's tests/bench and the CPU oracle's tests.

The paper's datasets (Evrard collapse and square patch snapshots, P:389-390,
Table IV) are not available; these recipes stand in for them
(DESIGN.md section 5):

  cfg 1  N=10,000 uniform [0,1)^3, constant h=0.0668
  cfg 2  N=1e6 uniform [0,1)^3, h_i = 0.0144 * U(0.8, 1.2)
  cfg 3  100^3 lattice at (i+0.5)*0.01 + N(0, 0.001^2) jitter, h = 0.015   (SP-like)
  cfg 4  N=4e6 Evrard-like sphere, density ~ 1/r inside R=1, h from n(r)  (EC-like)
  cfg 5  N=2^25: half uniform, half in 64 Gaussian clumps (sigma 0.01),
         h from a 64^3 histogram density estimate (target ~100 neighbors)

Generator: numpy PCG64 ``default_rng(1234 + cfg)``, draws in the order listed,
then a seeded random permutation of particle order (input order carries no
spatial locality).  ``n`` overrides the particle count for scaled-down parity
cases; h is rescaled as n^(-1/3) so the neighbor count stays ~100.
"""
from __future__ import annotations

import numpy as np

FULL_N = {1: 10_000, 2: 1_000_000, 3: 1_000_000, 4: 4_000_000, 5: 1 << 25}
BUCKET_SIZE = 64
MAX_EMPTY = 0.5
NGMAX = 512
TARGET_NEIGHBORS = 100.0


def _finish(rng, pos, h):
    perm = rng.permutation(pos.shape[0])
    pos = np.ascontiguousarray(pos[perm], dtype=np.float64)
    h = np.ascontiguousarray(h[perm], dtype=np.float64)
    return pos, h


def make_config(cfg: int, n: int | None = None, seed_offset: int = 0):
    """Return (pos float64 [N,3] C-contiguous, h float64 [N]) for config cfg."""
    if cfg not in FULL_N:
        raise ValueError(f"unknown config {cfg}")
    N = FULL_N[cfg] if n is None else int(n)
    rng = np.random.default_rng(1234 + cfg + 1000 * seed_offset)
    scale = (FULL_N[cfg] / max(N, 1)) ** (1.0 / 3.0)
    if cfg == 1:
        pos = rng.random((N, 3))
        h = np.full(N, 0.0668 * scale)
    elif cfg == 2:
        pos = rng.random((N, 3))
        h = 0.0144 * scale * rng.uniform(0.8, 1.2, N)
    elif cfg == 3:
        m = max(1, int(round(N ** (1.0 / 3.0))))
        N = m ** 3
        a = 1.0 / m
        g = (np.arange(m) + 0.5) * a
        gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
        pos = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
        pos = pos + rng.normal(0.0, 0.1 * a, size=(N, 3))
        h = np.full(N, 1.5 * a)
    elif cfg == 4:
        r = np.sqrt(rng.random(N))
        d = rng.normal(size=(N, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pos = d * r[:, None]
        # n(r) = N / (2 pi R^2 r); (4/3) pi (2h)^3 n = 100  =>  h = 1/2 (150 r / N)^(1/3)
        h = 0.5 * np.cbrt(150.0 * r / N)
        h = np.maximum(h, 1e-6)
    else:  # cfg 5
        nu = N // 2
        nc = N - nu
        uni = rng.random((nu, 3))
        centers = rng.random((64, 3))
        which = rng.integers(0, 64, nc)
        clump = centers[which] + rng.normal(0.0, 0.01, size=(nc, 3))
        pos = np.concatenate([uni, clump], axis=0)
        G = 64
        cell = np.clip(np.floor(pos * G).astype(np.int64), 0, G - 1)
        flat = (cell[:, 0] * G + cell[:, 1]) * G + cell[:, 2]
        counts = np.bincount(flat, minlength=G ** 3)
        nbin = counts[flat].astype(np.float64) * G ** 3
        h = 0.5 * np.cbrt(3.0 * TARGET_NEIGHBORS / (4.0 * np.pi * nbin))
    return _finish(rng, pos, h)


# ---- small structured cases for pins and edge cases --------------------------

def lattice(m: int, a: float = 1.0, origin: float = 0.0):
    """m^3 integer lattice with spacing a (coordinates exact in fp64 for a = 1)."""
    g = origin + a * np.arange(m, dtype=np.float64)
    gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
    return np.ascontiguousarray(np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1))


def uniform(n: int, seed: int, h_lo: float, h_hi: float | None = None, box: float = 1.0):
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3)) * box
    if h_hi is None:
        h = np.full(n, h_lo)
    else:
        h = rng.uniform(h_lo, h_hi, n)
    return np.ascontiguousarray(pos), np.ascontiguousarray(h)


def clustered(n: int, seed: int, nclumps: int = 8, sigma: float = 0.02, frac: float = 0.7,
              h: float = 0.03):
    """Mixture of Gaussian clumps and a uniform background (non-uniform trees)."""
    rng = np.random.default_rng(seed)
    nc = int(n * frac)
    centers = rng.random((nclumps, 3))
    which = rng.integers(0, nclumps, nc)
    pos = np.concatenate([centers[which] + rng.normal(0, sigma, (nc, 3)),
                          rng.random((n - nc, 3))], axis=0)
    hh = h * rng.uniform(0.5, 1.5, n)
    perm = rng.permutation(n)
    return np.ascontiguousarray(pos[perm]), np.ascontiguousarray(hh[perm])


def near_boundary(groups: int, partners: int, seed: int):
    """Adversarial set ("cfg 0"): each group is a query particle plus `partners`
    particles placed at distance 2h (1 + k 2^-52), k in [-8, 8], along random
    and axis-aligned directions, so that many pairs sit within a few ulps of the
    strict threshold.  All particles of a group share h (the gather criterion
    then tests both directions near the boundary).  A further 1/8 of the
    particles are snapped to dyadic and 1/b grids so they sit on sub-cell faces.
    """
    rng = np.random.default_rng(seed)
    pts = []
    hs = []
    for g in range(groups):
        c = rng.random(3)
        hg = rng.uniform(0.002, 0.02)
        t = 2.0 * hg
        pts.append(c)
        hs.append(hg)
        for p in range(partners):
            k = int(rng.integers(-8, 9))
            if p % 4 == 0:
                d = np.zeros(3)
                d[p % 3] = 1.0 if (p // 4) % 2 == 0 else -1.0
            else:
                d = rng.normal(size=3)
                d /= np.linalg.norm(d)
            r = t * (1.0 + k * 2.0 ** -52)
            pts.append(c + d * r)
            hs.append(hg)
    pos = np.array(pts, dtype=np.float64)
    h = np.array(hs, dtype=np.float64)
    nsnap = pos.shape[0] // 8
    sel = rng.choice(pos.shape[0], nsnap, replace=False)
    grids = np.array([64.0, 6.0, 25.0, 40.0, 81.0, 2.0, 3.0])
    gsel = grids[rng.integers(0, grids.size, nsnap)]
    pos[sel] = np.round(pos[sel] * gsel[:, None]) / gsel[:, None]
    perm = rng.permutation(pos.shape[0])
    return np.ascontiguousarray(pos[perm]), np.ascontiguousarray(h[perm])
