"""UPGMA guide tree — ORACLE (test infrastructure only).

SPEC S:356-364 `upgma(matrix) -> GuideTree`: "standard UPGMA: repeatedly merge the closest pair
under average linkage; ties broken by smallest (i,j) lexicographic index (decision D-M1)". The
guide-tree stage of the per-bucket aligner ("The k-mer distance can be used to
rapidly construct phylogenetic trees", step 7).

Plain and slow (numpy, O(n^3)). Conventions (shared by the GPU kernel by definition, not by code):
  * a cluster lives at the position of its smallest leaf; leaves are 0..n-1, the cluster made by
    step t gets id n + t (scipy's linkage numbering);
  * step t merges the active positions i < j with the smallest d(i, j), ties -> smallest i, then
    smallest j (row-major order of the upper triangle);
  * the join height is d(i, j) / 2;
  * average linkage: d(k, i u j) = (n_i d(k, i) + n_j d(k, j)) / (n_i + n_j), evaluated in IEEE
    float64 as the rounded products, their rounded sum, then the rounded quotient (no FMA).
Input: the k-mer distance d_ij = 1 - S_ij / den_ij in float64 (rounded division, rounded subtraction).
"""
from __future__ import annotations

import numpy as np


def distance_f64(S, den) -> np.ndarray:
    """d = 1 - S/den (float64, IEEE), 0 on the diagonal."""
    d = np.float64(1.0) - np.asarray(S, dtype=np.float64) / np.asarray(den, dtype=np.float64)
    np.fill_diagonal(d, 0.0)
    return d


def upgma(D):
    """Returns (merges int64 [n-1, 2] of cluster ids (id at position i, id at position j),
    heights float64 [n-1], sizes int64 [n-1])."""
    D = np.array(D, dtype=np.float64, copy=True)
    n = D.shape[0]
    active = np.ones(n, bool)
    size = np.ones(n, np.int64)
    cid = np.arange(n, dtype=np.int64)
    merges = np.zeros((max(n - 1, 0), 2), np.int64)
    heights = np.zeros(max(n - 1, 0), np.float64)
    sizes = np.zeros(max(n - 1, 0), np.int64)
    iu = np.triu(np.ones((n, n), bool), 1)
    for t in range(n - 1):
        mask = iu & active[:, None] & active[None, :]
        flat = np.where(mask, D, np.inf).ravel()
        x = int(np.argmin(flat))                      # first minimum in row-major order: smallest (i, j)
        i, j = divmod(x, n)
        merges[t] = (cid[i], cid[j])
        heights[t] = D[i, j] / 2.0
        ni, nj = np.float64(size[i]), np.float64(size[j])
        new = (ni * D[i] + nj * D[j]) / (ni + nj)     # each op rounded once (numpy: no FMA)
        D[i, :] = new
        D[:, i] = new
        D[i, i] = 0.0
        size[i] += size[j]
        sizes[t] = size[i]
        active[j] = False
        cid[i] = n + t
    return merges, heights, sizes
