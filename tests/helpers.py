"""Seeded synthetic data for parity tests (numpy only)."""

import numpy as np


def mixture(rng, n, d, comps=256, hi=128.0, sigma=16.0, clip=(0.0, 255.0)):
    """BASELINE cfg0 family: isotropic Gaussian mixture, centres U[0,hi]."""
    centers = rng.uniform(0.0, hi, size=(comps, d)).astype(np.float32)
    lab = rng.integers(0, comps, size=n)
    x = centers[lab] + rng.normal(0.0, sigma, size=(n, d)).astype(np.float32)
    if clip is not None:
        x = np.clip(x, clip[0], clip[1])
    return x.astype(np.float32)


def kmeans_books(x, m, k, iters=4, seed=0):
    """Small per-sub-space Lloyd k-means (test data prep only)."""
    rng = np.random.default_rng(seed)
    n, d = x.shape
    dsub = d // m
    books = np.empty((m, k, dsub), np.float32)
    for j in range(m):
        sub = x[:, j * dsub:(j + 1) * dsub].astype(np.float32)
        c = sub[rng.choice(n, k, replace=False)].copy()
        for _ in range(iters):
            dd = (sub * sub).sum(1)[:, None] - 2 * sub @ c.T + (c * c).sum(1)[None]
            a = dd.argmin(1)
            for t in range(k):
                sel = a == t
                if sel.any():
                    c[t] = sub[sel].mean(0)
        books[j] = c
    return books


def encode(books, x, chunk=65536):
    m, k, dsub = books.shape
    out = np.empty((x.shape[0], m), np.uint8)
    for lo in range(0, x.shape[0], chunk):
        xs = x[lo:lo + chunk]
        for j in range(m):
            sub = xs[:, j * dsub:(j + 1) * dsub]
            c = books[j]
            dd = (sub * sub).sum(1)[:, None] - 2 * sub @ c.T + (c * c).sum(1)[None]
            out[lo:lo + chunk, j] = dd.argmin(1)
    return out
