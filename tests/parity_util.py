"""Shared helpers for GPU-vs-oracle parity tests: tolerances of SURVEY.md 8(c) and layout conversions."""
import numpy as np

import oracle as O

# north_star tolerances (FP32 accumulation); FP64 mode: 1e-10 on C
TOL_C, TOL_G, TOL_H = 1e-4, 1e-3, 1e-3
TOL_ROT_DEG, TOL_SHIFT = 0.05, 0.1


def c_tol(C_ref, E, fp64=False):
    return (1e-10 if fp64 else TOL_C) * max(abs(C_ref), 1e-2 * E)


def g_tol(g_ref, E, L, fp64=False):
    return (1e-9 if fp64 else TOL_G) * max(np.abs(g_ref).max(), 1e-2 * (1 + L) * E)


def h_tol(h_ref, E, L, fp64=False):
    return (1e-9 if fp64 else TOL_H) * max(np.abs(h_ref).max(), 1e-2 * (1 + L) ** 2 * E)


def rot_err_deg(e1, e2):
    return O.geodesic_deg(e1, e2)


def topk_index_must_match(all_scores, all_idx, k, grid, E0):
    """SURVEY 8(c) top-K rule: rank k is compared only if its score is separated by > 1e-4 E_{L0} from ranks
    k-1, k+1 (incl. the best unselected maximum) and no grid neighbour is within 1e-4 E_{L0} of it."""
    tol = 1e-4 * E0
    s = all_scores
    if k >= len(s):
        return False
    if k > 0 and abs(s[k - 1] - s[k]) <= tol:
        return False
    if k + 1 < len(s) and abs(s[k] - s[k + 1]) <= tol:
        return False
    nb, na, ng = grid.shape
    i = int(all_idx[k])
    j, a, c = i // (na * ng), (i // ng) % na, i % ng
    v = grid[j, a, c]
    for dj in (-1, 0, 1):
        if not 0 <= j + dj < nb:
            continue
        for da in (-1, 0, 1):
            for dc in (-1, 0, 1):
                if dj == da == dc == 0:
                    continue
                if abs(grid[j + dj, (a + da) % na, (c + dc) % ng] - v) <= tol:
                    return False
    return True
