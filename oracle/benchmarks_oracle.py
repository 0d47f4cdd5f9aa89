"""TEST INFRASTRUCTURE ONLY -- numpy oracles of the five tunable benchmark
kernels (paper_2102_05297_b200/kernels/*.cu).  Only tests/ may import this
module, as the checker of the CUDA outputs; nothing on the product path
reads it.

The reference ships no benchmark kernels and no oracles for them (SURVEY
section 0.2 item 3): each function restates the kernel's mathematical
definition in float64 and also returns the magnitude sum of the terms, so that
tests can state an FP32 tolerance relative to sum |term| (a sum with
cancellation has no meaningful element-wise relative error).

    coulomb   PAPER.md:84-89 (Eq. 1) with w_j = q_j / (4 pi eps0) folded in
    transpose out[x][y] = in[y][x]
    gemm      C = A B, A given K-major (AT[K][M])
    nbody     a_i = sum_j m_j d_ij / (|d_ij|^2 + eps^2)^(3/2)
    conv      zero-padded FILTER x FILTER correlation (out[y][x] =
              sum in[y + fy - R][x + fx - R] f[fy][fx])
"""

import numpy as np


def transpose(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a.T)


def coulomb(atoms: np.ndarray, spacing: float, grid: int):
    """atoms: (n, 4) float32 x, y, z, w.  Returns (V, sum |w|/r) on the
    (z, y, x) grid, float64."""
    a = atoms.astype(np.float64)
    coords = np.arange(grid, dtype=np.float64) * np.float64(np.float32(spacing))
    v = np.zeros((grid, grid, grid))
    mag = np.zeros((grid, grid, grid))
    zz, yy, xx = np.meshgrid(coords, coords, coords, indexing="ij")
    for x, y, z, w in a:
        r = np.sqrt((xx - x) ** 2 + (yy - y) ** 2 + (zz - z) ** 2)
        v += w / r
        mag += abs(w) / r
    return v, mag


def gemm(at: np.ndarray, b: np.ndarray):
    """at: (K, M), b: (K, N).  Returns (C, |A| |B|) in float64."""
    a = at.astype(np.float64).T
    bb = b.astype(np.float64)
    return a @ bb, np.abs(a) @ np.abs(bb)


def nbody(pm: np.ndarray, eps2: float):
    """pm: (n, 4) float32 x, y, z, m.  Returns (acc (n, 3), magnitude (n, 3))."""
    p = pm[:, :3].astype(np.float64)
    m = pm[:, 3].astype(np.float64)
    acc = np.zeros_like(p)
    mag = np.zeros_like(p)
    for s in range(0, p.shape[0], 1024):
        d = p[None, :, :] - p[s:s + 1024, None, :]           # (blk, n, 3)
        r2 = (d * d).sum(axis=2) + np.float64(np.float32(eps2))
        inv3 = r2 ** -1.5
        t = d * (m[None, :] * inv3)[:, :, None]
        acc[s:s + 1024] = t.sum(axis=1)
        mag[s:s + 1024] = np.abs(t).sum(axis=1)
    return acc, mag


def conv(img: np.ndarray, filt: np.ndarray):
    """img: (H, W), filt: (F, F).  Returns (out, sum |in f|) in float64."""
    f = filt.shape[0]
    r = f // 2
    x = np.pad(img.astype(np.float64), r)
    h, w = img.shape
    out = np.zeros((h, w))
    mag = np.zeros((h, w))
    ff = filt.astype(np.float64)
    for fy in range(f):
        for fx in range(f):
            t = x[fy:fy + h, fx:fx + w] * ff[fy, fx]
            out += t
            mag += np.abs(t)
    return out, mag


def within(got: np.ndarray, want: np.ndarray, mag: np.ndarray, rtol: float) -> float:
    """Largest |got - want| / (mag + tiny) -- the relative error against the
    magnitude sum of the terms; a test asserts it is <= rtol."""
    err = np.abs(got.astype(np.float64) - want) / (mag + 1e-30)
    return float(err.max()) if err.size else 0.0
