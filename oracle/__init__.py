"""FP64 CPU oracle for the Matcha hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2603_15285_b200``) never imports it.  It wraps ``oracle/liboracle.so``
(``oracle/oracle.cpp``), which shares no code with the CUDA library.

Layouts (numpy):
  F, H     complex128 [ncoef(L), R]  (lm = l(l+1)/2 + m, m >= 0; unweighted shell coefficients)
  M full   complex128 flat, blocks l = 0..Lc of (2l+1) x (2l+1), entry (m+l)(2l+1) + (n+l)
  M half   complex128 [Mh(L)]: (l, m in [0,l], n in [-l,l]) at l(l+1)(4l-1)/6 + m(2l+1) + (n+l)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_d = ctypes.c_double
_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int)
_i64p = ctypes.POINTER(ctypes.c_int64)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle`")
        lib = ctypes.CDLL(path)
        sig = {
            "orc_euler_to_matrix": [_dp, _dp],
            "orc_matrix_to_euler": [_dp, _dp],
            "orc_canon": [_dp],
            "orc_gauss_legendre": [ctypes.c_int, _dp, _dp],
            "orc_legendre_norm": [ctypes.c_int, _d, _dp],
            "orc_wigner_d": [ctypes.c_int, _d, _dp, _dp, _dp],
            "orc_sh_analysis_vol": [_fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp],
            "orc_sh_analysis_poly": [_dp, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp],
            "orc_sh_analysis_batch": [_fp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp,
                                      ctypes.c_int],
            "orc_corr_full": [_dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp],
            "orc_eval_corr": [_dp, ctypes.c_int, _dp, _dp],
            "orc_grid_eval": [_dp, ctypes.c_int, ctypes.c_int, _dp],
            "orc_find_maxima": [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _dp],
            "orc_grid_node_euler": [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _dp],
            "orc_newton_delta": [_dp, _dp, _dp],
            "orc_refine": [_dp, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _d, _d, _d, _dp, _dp, _ip],
            "orc_rotate_volume": [_fp, ctypes.c_int, _dp, _dp],
            "orc_translation": [_fp, _fp, ctypes.c_int, _dp, ctypes.c_int, _dp, _dp],
            "orc_translation_upsampled": [_fp, _fp, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp],
            "orc_upsampled_corr_at": [_fp, _fp, ctypes.c_int, _dp, _dp],
            "orc_energy": [_dp, _dp, ctypes.c_int, ctypes.c_int],
            "orc_align_batch": [_fp, ctypes.c_int64, _fp, _dp, ctypes.c_int, _ip, _dp, _dp, ctypes.c_int],
            "orc_align_batch_multi": [_fp, ctypes.c_int64, _fp, ctypes.c_int, _dp, ctypes.c_int, _ip, _dp, _dp,
                                      ctypes.c_int],
            "orc_ball_tables": [ctypes.c_int, ctypes.c_int, _d, _ip, _dp],
            "orc_sph_bessel": [ctypes.c_int, _d],
            "orc_ball_transform": [_dp, ctypes.c_int, ctypes.c_int, _d, _dp],
            "orc_corr_ball_full": [_dp, _dp, ctypes.c_int, ctypes.c_int, _d, ctypes.c_int, _dp],
            "orc_reconstruct": [_fp, ctypes.c_int64, ctypes.c_int, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int64, _dp, _ip],
        }
        for name, args in sig.items():
            getattr(lib, name).argtypes = args
        lib.orc_find_maxima.restype = ctypes.c_int
        lib.orc_energy.restype = ctypes.c_double
        lib.orc_upsampled_corr_at.restype = ctypes.c_double
        lib.orc_ball_tables.restype = ctypes.c_int
        lib.orc_sph_bessel.restype = ctypes.c_double
        _LIB = lib
    return _LIB


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _c128(a):
    return np.ascontiguousarray(a, np.complex128)


# ---------------------------------------------------------------- sizes / layouts
def ncoef(L):
    return (L + 1) * (L + 2) // 2


def full_size(L):
    return sum((2 * l + 1) ** 2 for l in range(L + 1))


def full_offset(l):
    return l * (2 * l - 1) * (2 * l + 1) // 3


def half_size(L):
    return (L + 1) * (L + 2) * (4 * L + 3) // 6


def half_offset(l):
    return l * (l + 1) * (4 * l - 1) // 6


def grid_dims(L0, K):
    return K * (L0 + 1), 2 * K * (L0 + 1), 2 * K * (L0 + 1)


def full_to_half(Mf, L):
    out = np.empty(half_size(L), np.complex128)
    for l in range(L + 1):
        w = 2 * l + 1
        blk = Mf[full_offset(l):full_offset(l) + w * w].reshape(w, w)
        out[half_offset(l):half_offset(l) + (l + 1) * w] = blk[l:, :].reshape(-1)
    return out


def half_to_full(Mh, L):
    """Rebuild the full plane from the half plane via M_{-m,-n} = (-1)^{m+n} conj M_{mn} (real inputs)."""
    out = np.empty(full_size(L), np.complex128)
    for l in range(L + 1):
        w = 2 * l + 1
        top = Mh[half_offset(l):half_offset(l) + (l + 1) * w].reshape(l + 1, w)
        blk = np.empty((w, w), np.complex128)
        blk[l:, :] = top
        for m in range(1, l + 1):
            for n in range(-l, l + 1):
                blk[-m + l, -n + l] = (-1) ** ((m + n) & 1) * np.conj(top[m, n + l])
        out[full_offset(l):full_offset(l) + w * w] = blk.reshape(-1)
    return out


# ---------------------------------------------------------------- primitives
def euler_to_matrix(e):
    R = np.zeros(9)
    _lib().orc_euler_to_matrix(_p(np.ascontiguousarray(e, np.float64)), _p(R))
    return R.reshape(3, 3)


def matrix_to_euler(R):
    e = np.zeros(3)
    _lib().orc_matrix_to_euler(_p(np.ascontiguousarray(R, np.float64).reshape(9)), _p(e))
    return e


def canon(e):
    e = np.array(e, np.float64)
    _lib().orc_canon(_p(e))
    return e


def geodesic_deg(e1, e2):
    R1, R2 = euler_to_matrix(e1), euler_to_matrix(e2)
    return geodesic_deg_matrix(R1, R2)


def geodesic_deg_matrix(R1, R2):
    """Geodesic angle acos((tr(R1^T R2) - 1)/2), evaluated as atan2(sin, cos) for accuracy near 0."""
    Q = np.asarray(R1).T @ np.asarray(R2)
    c = (np.trace(Q) - 1.0) / 2.0
    s = 0.5 * np.sqrt((Q[2, 1] - Q[1, 2]) ** 2 + (Q[0, 2] - Q[2, 0]) ** 2 + (Q[1, 0] - Q[0, 1]) ** 2)
    return float(np.degrees(np.arctan2(s, c)))


def gauss_legendre(n):
    x, w = np.zeros(n), np.zeros(n)
    _lib().orc_gauss_legendre(n, _p(x), _p(w))
    return x, w


def legendre_norm(L, x):
    P = np.zeros(ncoef(L))
    _lib().orc_legendre_norm(L, x, _p(P))
    return P


def wigner_d(l, beta, derivs=False):
    w = 2 * l + 1
    d, d1, d2 = np.zeros(w * w), np.zeros(w * w), np.zeros(w * w)
    _lib().orc_wigner_d(l, beta, _p(d), _p(d1) if derivs else None, _p(d2) if derivs else None)
    if derivs:
        return d.reshape(w, w), d1.reshape(w, w), d2.reshape(w, w)
    return d.reshape(w, w)


def wigner_D(l, e):
    d = wigner_d(l, e[1])
    m = np.arange(-l, l + 1)
    return np.exp(-1j * m[:, None] * e[0]) * d * np.exp(-1j * m[None, :] * e[2])


# ---------------------------------------------------------------- stages
def sh_analysis(vol, L, qover=2, shift=None):
    vol = np.ascontiguousarray(vol, np.float32)
    N = vol.shape[-1]
    F = np.zeros((ncoef(L), N // 2), np.complex128)
    sh = None if shift is None else np.ascontiguousarray(shift, np.float64)
    _lib().orc_sh_analysis_vol(_p(vol, _fp), N, L, qover, _p(sh), _p(F.view(np.float64)))
    return F


def sh_analysis_batch(vols, L, qover=2, shifts=None, nthreads=0):
    vols = np.ascontiguousarray(vols, np.float32)
    B, N = vols.shape[0], vols.shape[-1]
    F = np.zeros((B, ncoef(L), N // 2), np.complex128)
    sh = None if shifts is None else np.ascontiguousarray(shifts, np.float64)
    _lib().orc_sh_analysis_batch(_p(vols, _fp), B, N, L, qover, _p(sh), _p(F.view(np.float64)), nthreads)
    return F


def sh_analysis_poly(terms, N, L, qover=2, R=None):
    """terms: list of (coef, a, b, c) for u(y) = sum coef y_x^a y_y^b y_z^c, sampled at y = R^T(p - c)."""
    t = np.ascontiguousarray(np.array(terms, np.float64).reshape(-1, 4))
    Rm = None if R is None else np.ascontiguousarray(R, np.float64).reshape(9)
    F = np.zeros((ncoef(L), N // 2), np.complex128)
    _lib().orc_sh_analysis_poly(_p(t), t.shape[0], _p(Rm), N, L, qover, _p(F.view(np.float64)))
    return F


def corr_full(F, H, Lc):
    F, H = _c128(F), _c128(H)
    L = int(round((np.sqrt(8 * F.shape[0] + 1) - 3) / 2))
    M = np.zeros(full_size(Lc), np.complex128)
    _lib().orc_corr_full(_p(F.view(np.float64)), _p(H.view(np.float64)), L, Lc, F.shape[1], _p(M.view(np.float64)))
    return M


def eval_corr(Mf, L, e):
    """-> (C, grad[3] (a,b,g), hess[6] (aa,bb,gg,ab,ag,bg)) of C_L at Euler angles e."""
    out = np.zeros(10)
    _lib().orc_eval_corr(_p(_c128(Mf).view(np.float64)), L, _p(np.ascontiguousarray(e, np.float64)), _p(out))
    return out[0], out[1:4].copy(), out[4:10].copy()


def grid_eval(Mf, L0, K):
    nb, na, ng = grid_dims(L0, K)
    g = np.zeros((nb, na, ng))
    _lib().orc_grid_eval(_p(_c128(Mf).view(np.float64)), L0, K, _p(g))
    return g


def find_maxima(grid, ncand):
    grid = np.ascontiguousarray(grid, np.float64)
    idx = np.zeros(ncand, np.int64)
    sc = np.zeros(ncand)
    n = _lib().orc_find_maxima(_p(grid), grid.shape[0], grid.shape[1], grid.shape[2], ncand, _p(idx, _i64p), _p(sc))
    return idx, sc, n


def grid_node_euler(idx, L0, K):
    e = np.zeros(3)
    _lib().orc_grid_node_euler(int(idx), L0, K, _p(e))
    return e


def newton_delta(g, h):
    dl = np.zeros(3)
    _lib().orc_newton_delta(_p(np.ascontiguousarray(g, np.float64)), _p(np.ascontiguousarray(h, np.float64)),
                            _p(dl))
    return dl


def refine(Mf, bands, iters, euler, idx=None, tols=(0.0, 0.0, 0.0)):
    eu = np.array(euler, np.float64).reshape(-1, 3).copy()
    nc = eu.shape[0]
    b = np.ascontiguousarray(bands, np.int32)
    sc = np.zeros(nc)
    best = ctypes.c_int(-1)
    ix = None if idx is None else np.ascontiguousarray(idx, np.int64)
    _lib().orc_refine(_p(_c128(Mf).view(np.float64)), _p(b, _ip), len(b), iters, nc, _p(ix, _i64p), tols[0],
                      tols[1], tols[2], _p(eu), _p(sc), ctypes.byref(best))
    return eu, sc, best.value


def rotate_volume(ref, e):
    ref = np.ascontiguousarray(ref, np.float32)
    out = np.zeros(ref.shape, np.float64)
    _lib().orc_rotate_volume(_p(ref, _fp), ref.shape[-1], _p(np.ascontiguousarray(e, np.float64)), _p(out))
    return out


def translation(vol, ref, e, W):
    vol = np.ascontiguousarray(vol, np.float32)
    ref = np.ascontiguousarray(ref, np.float32)
    sh, pk = np.zeros(3), np.zeros(1)
    _lib().orc_translation(_p(vol, _fp), _p(ref, _fp), vol.shape[-1], _p(np.ascontiguousarray(e, np.float64)), W,
                           _p(sh), _p(pk))
    return sh, float(pk[0])


def translation_upsampled(vol, ref, e, W, kappa=16):
    """Integer windowed peak, then the upsampled-DFT refinement (Guizar-Sicairos; App. C remark iii)."""
    vol = np.ascontiguousarray(vol, np.float32)
    ref = np.ascontiguousarray(ref, np.float32)
    sh, pk = np.zeros(3), np.zeros(1)
    _lib().orc_translation_upsampled(_p(vol, _fp), _p(ref, _fp), vol.shape[-1],
                                     _p(np.ascontiguousarray(e, np.float64)), W, kappa, _p(sh), _p(pk))
    return sh, float(pk[0])


def upsampled_corr_at(vol, ref, e, t):
    """c~(t) = (1/N^3) Re sum_k F^ conj(rho^) D(kx,tx) D(ky,ty) D(kz,tz) at one point (full triple sum; D(k,t) =
    e^{2 pi i k' t/N}, k' the symmetric frequency, D(N/2, t) = cos(pi t): reading C27)."""
    vol = np.ascontiguousarray(vol, np.float32)
    ref = np.ascontiguousarray(ref, np.float32)
    return _lib().orc_upsampled_corr_at(_p(vol, _fp), _p(ref, _fp), vol.shape[-1],
                                        _p(np.ascontiguousarray(e, np.float64)),
                                        _p(np.ascontiguousarray(t, np.float64)))


def energy(F, H, Lc):
    F, H = _c128(F), _c128(H)
    return _lib().orc_energy(_p(F.view(np.float64)), _p(H.view(np.float64)), Lc, F.shape[1])


def align_batch(vols, ref, params, H=None, nthreads=0):
    """params: dict with L, qover, L0, K, ncand, bands, iters, T, W, ups (0: parabolic subpixel, kappa: upsampled
    DFT), tol_grad, tol_step, tol_obj.
    -> poses [B, 8] = (alpha, beta, gamma, tx, ty, tz, score, best)."""
    vols = np.ascontiguousarray(vols, np.float32)
    ref = np.ascontiguousarray(ref, np.float32)
    B, N = vols.shape[0], vols.shape[-1]
    bands = list(params["bands"])
    ip, dp = _param_arrays(params)
    Hc = None if H is None else _c128(H)
    poses = np.zeros((B, 8))
    _lib().orc_align_batch(_p(vols, _fp), B, _p(ref, _fp), None if Hc is None else _p(Hc.view(np.float64)), N,
                           _p(ip, _ip), _p(dp), _p(poses), nthreads)
    return poses


def _param_arrays(params):
    bands = list(params["bands"])
    ip = np.zeros(27, np.int32)
    ip[0:6] = [params["L"], params.get("qover", 2), params["L0"], params.get("K", 2), params["ncand"], len(bands)]
    ip[6:6 + len(bands)] = bands
    ip[22:27] = [params.get("iters", 1), params.get("T", 1), params.get("W", 0), params.get("ups", 0),
                 params.get("radial", 0)]
    dp = np.array([params.get("tol_grad", 0.0), params.get("tol_step", 0.0), params.get("tol_obj", 0.0),
                   params.get("lam", 0.0)])
    return ip, dp


def align_batch_multi(vols, refs, params, nthreads=0):
    """Multi-template alignment: refs [T, N, N, N] -> poses [B, 9] (..., template index)."""
    vols = np.ascontiguousarray(vols, np.float32)
    refs = np.ascontiguousarray(refs, np.float32)
    B, N = vols.shape[0], vols.shape[-1]
    ip, dp = _param_arrays(params)
    poses = np.zeros((B, 9))
    _lib().orc_align_batch_multi(_p(vols, _fp), B, _p(refs, _fp), refs.shape[0], None, N, _p(ip, _ip), _p(dp),
                                 _p(poses), nthreads)
    return poses


def reconstruct(vols, poses, n_classes=1, class_col=-1, first_index=0):
    """Half-map sums: -> (sums [n_classes, 2, N, N, N], counts [n_classes, 2])."""
    vols = np.ascontiguousarray(vols, np.float32)
    poses = np.ascontiguousarray(poses, np.float64)
    B, N = vols.shape[0], vols.shape[-1]
    sums = np.zeros((n_classes, 2, N, N, N))
    counts = np.zeros((n_classes, 2), np.int32)
    _lib().orc_reconstruct(_p(vols, _fp), B, N, _p(poses), poses.shape[1], class_col, n_classes, first_index,
                           _p(sums), _p(counts, _ip))
    return sums, counts


# ---------------------------------------------------------------- ball-harmonic radial basis
def ball_tables(L, R, lam=0.0):
    """-> (K [L+1] = |K_l|, Bt [L+1, Kmax, R] radial weights (1/R) rho_i^2 c_lk j_l(lambda_lk rho_i))."""
    K = np.zeros(L + 1, np.int32)
    Kmax = _lib().orc_ball_tables(L, R, lam, _p(K, _ip), None)
    Bt = np.zeros((L + 1, Kmax, R))
    _lib().orc_ball_tables(L, R, lam, _p(K, _ip), _p(Bt))
    return K, Bt


def sph_bessel(l, x):
    return _lib().orc_sph_bessel(l, float(x))


def ball_transform(F, lam=0.0):
    F = _c128(F)
    L = int(round((np.sqrt(8 * F.shape[0] + 1) - 3) / 2))
    R = F.shape[1]
    K, _ = ball_tables(L, R, lam)
    Fb = np.zeros((F.shape[0], int(K.max())), np.complex128)
    _lib().orc_ball_transform(_p(F.view(np.float64)), L, R, lam, _p(Fb.view(np.float64)))
    return Fb


def corr_ball_full(Fb, Hb, R, Lc, lam=0.0):
    Fb, Hb = _c128(Fb), _c128(Hb)
    L = int(round((np.sqrt(8 * Fb.shape[0] + 1) - 3) / 2))
    M = np.zeros(full_size(Lc), np.complex128)
    _lib().orc_corr_ball_full(_p(Fb.view(np.float64)), _p(Hb.view(np.float64)), L, R, lam, Lc, _p(M.view(np.float64)))
    return M
