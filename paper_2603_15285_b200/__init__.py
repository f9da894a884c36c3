"""paper_2603_15285_b200 -- B200-native (sm_100a) hot path of Matcha (arXiv 2603.15285).

Thin Python binding over the C ABI of ``libmatcha.so`` (``include/matcha.h``): argument
marshalling only.  Every step of the path runs in the library's CUDA kernels; torch is used
for device memory and streams.  There is no CPU fallback: importing this package without the
built library raises.

    h = Handle(N=64, L_max=32)
    poses = h.align_batch(vols, ref, Params(bands=(8, 12, 16, 24, 32)))   # [B, 8]
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmatcha.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make cuda` (or __graft_entry__.build()); "
                      "the Matcha hot path has no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

MATCHA_OK = 0
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "DEGREE", -3: "CUTOFF", -4: "SHAPE", -5: "WINDOW", -6: "NONFINITE",
          -7: "CUDA", -8: "ALLOC", -9: "NOT_IMPLEMENTED", -10: "OVERFLOW"}
FP32, FP64 = 0, 1


class MatchaError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"matcha {STATUS.get(status, status)} ({status}): {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int32), ("L_max", ctypes.c_int32), ("quad_oversample", ctypes.c_int32),
                ("max_batch", ctypes.c_int32), ("precision", ctypes.c_int32)]


class _Params(ctypes.Structure):
    _fields_ = [("n_bands", ctypes.c_int32), ("bands", ctypes.c_int32 * 16), ("newton_iters", ctypes.c_int32),
                ("n_cand", ctypes.c_int32), ("oversample", ctypes.c_int32), ("n_alternations", ctypes.c_int32),
                ("shift_window", ctypes.c_int32), ("upsample", ctypes.c_int32), ("radial", ctypes.c_int32),
                ("tol_grad", ctypes.c_double), ("tol_step", ctypes.c_double), ("tol_obj", ctypes.c_double),
                ("ball_lambda", ctypes.c_double)]


_vp, _i64, _i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
_H = ctypes.c_void_p
_SIGS = {
    "matcha_create": ([ctypes.POINTER(_Config), ctypes.POINTER(_H)], ctypes.c_int),
    "matcha_destroy": ([_H], ctypes.c_int),
    "matcha_coeff_count": ([_H], ctypes.c_int64),
    "matcha_corr_count": ([_i32], ctypes.c_int64),
    "matcha_sh_analysis": ([_H, _vp, _i64, _vp, _vp, _vp], ctypes.c_int),
    "matcha_corr_coeffs": ([_H, _vp, _vp, _i64, _i32, _vp, _vp], ctypes.c_int),
    "matcha_so3_search": ([_H, _vp, _i32, _i64, _i32, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "matcha_eval_corr": ([_H, _vp, _i32, _i64, _i32, _i32, _vp, _vp, _vp, _vp, _vp], ctypes.c_int),
    "matcha_newton_refine": ([_H, _vp, _i32, _i64, _i32, ctypes.POINTER(_Params), _vp, _vp, _vp, _vp, _vp],
                             ctypes.c_int),
    "matcha_translation_update": ([_H, _vp, _i64, _vp, _vp, _i32, _i32, _vp, _vp, _vp], ctypes.c_int),
    "matcha_align_batch": ([_H, _vp, _i64, _vp, _vp, ctypes.POINTER(_Params), _vp, _vp], ctypes.c_int),
    "matcha_align_batch_host": ([_H, _vp, _i64, _vp, ctypes.POINTER(_Params), _vp, _vp], ctypes.c_int),
    "matcha_ball_kmax": ([_H, ctypes.c_double, ctypes.POINTER(ctypes.c_int32)], ctypes.c_int32),
    "matcha_ball_transform": ([_H, _vp, _i64, ctypes.c_double, _vp, _vp], ctypes.c_int),
    "matcha_corr_coeffs_ball": ([_H, _vp, _vp, _i64, _i32, ctypes.c_double, _vp, _vp], ctypes.c_int),
    "matcha_set_graphs": ([_H, _i32], ctypes.c_int),
    "matcha_synth_particles": ([_H, ctypes.c_uint64, _i64, _i64, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp],
                               ctypes.c_int),
    "matcha_align_multi": ([_H, _vp, _i64, _vp, _i32, _vp, ctypes.POINTER(_Params), _vp, _vp], ctypes.c_int),
    "matcha_reconstruct": ([_H, _vp, _i64, _vp, _i32, _i32, _i32, _i64, _vp, _vp, _vp], ctypes.c_int),
    "matcha_get_status": ([_H, _vp], ctypes.c_int),
    "matcha_last_error_string": ([_H], ctypes.c_char_p),
    "matcha_launch_count": ([_H], ctypes.c_int64),
    "matcha_profile_begin": ([_H], ctypes.c_int),
    "matcha_profile_end": ([_H, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
}
NUM_STAGES = 8
STAGES = ("sh_analysis", "corr_coeffs", "so3_search", "newton_refine", "gather_poses", "translation_update",
          "reconstruct", "ball_transform")
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def ncoef(L: int) -> int:
    return (L + 1) * (L + 2) // 2


def corr_count(L: int) -> int:
    """Mh(L) = (L+1)(L+2)(4L+3)/6 complex entries of the half-plane M."""
    return int(_lib.matcha_corr_count(L))


def half_offset(l: int) -> int:
    return l * (l + 1) * (4 * l - 1) // 6


@dataclass
class Params:
    """Algorithm 1 / App. C parameters (include/matcha.h matcha_params_t)."""
    bands: Sequence[int] = (8, 12, 16, 24, 32)
    newton_iters: int = 1
    n_cand: int = 10
    oversample: int = 2
    n_alternations: int = 1
    shift_window: int = 0
    upsample: int = 0          # 0: parabolic subpixel; kappa: upsampled-DFT subpixel
    radial: int = 0            # 0: shells; 1: ball harmonics with cutoff ball_lambda
    tol_grad: float = 0.0
    tol_step: float = 0.0
    tol_obj: float = 0.0
    ball_lambda: float = 0.0   # <= 0: pi (R - 1/2)

    def c(self) -> _Params:
        p = _Params()
        p.n_bands = len(self.bands)
        for i, b in enumerate(self.bands):
            p.bands[i] = int(b)
        p.newton_iters, p.n_cand, p.oversample = self.newton_iters, self.n_cand, self.oversample
        p.n_alternations, p.shift_window, p.upsample = self.n_alternations, self.shift_window, self.upsample
        p.tol_grad, p.tol_step, p.tol_obj = self.tol_grad, self.tol_step, self.tol_obj
        p.radial, p.ball_lambda = self.radial, self.ball_lambda
        return p


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Handle:
    """One handle per GPU (created on the current CUDA device)."""

    def __init__(self, N: int, L_max: int, quad_oversample: int = 2, max_batch: int = 1024,
                 precision: str = "fp32"):
        cfg = _Config(N, L_max, quad_oversample, max_batch, FP64 if precision == "fp64" else FP32)
        h = _H()
        self._check(_lib.matcha_create(ctypes.byref(cfg), ctypes.byref(h)), None)
        self._h = h
        self.N, self.L_max, self.R = N, L_max, N // 2
        self.max_batch = max_batch
        self.fp64 = precision == "fp64"
        self.real = torch.float64 if self.fp64 else torch.float32
        self.cplx = torch.complex128 if self.fp64 else torch.complex64
        self.device = torch.device("cuda", torch.cuda.current_device())

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:  # _lib is None during interpreter shutdown
            _lib.matcha_destroy(h)
            self._h = None

    def _arg(self, t: Optional[torch.Tensor], name: str, dtype, shape=None, optional: bool = False):
        """Validate a tensor argument before its pointer crosses the C ABI: the library reads raw bytes, so a wrong
        dtype (e.g. float64 angles handed to an FP32 handle), device, layout or shape would be reinterpreted
        silently.  Raises TypeError / ValueError; returns the tensor."""
        if t is None:
            if optional:
                return None
            raise ValueError(f"{name} is required")
        if not isinstance(t, torch.Tensor):
            raise TypeError(f"{name} must be a torch.Tensor, got {type(t).__name__}")
        if t.dtype != dtype:
            raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
        if not t.is_cuda or t.device != self.device:
            raise ValueError(f"{name} must live on {self.device}, got {t.device}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if shape is not None and tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
        return t

    def _check(self, st, h=None):
        if st != MATCHA_OK:
            msg = _lib.matcha_last_error_string(h if h is not None else self._h).decode() if (
                h is not None or getattr(self, "_h", None) is not None) else ""
            raise MatchaError(st, msg)

    def status(self):
        self._check(_lib.matcha_get_status(self._h, _stream()))

    @property
    def launches(self) -> int:
        return int(_lib.matcha_launch_count(self._h))

    def synth_particles(self, B: int, snr: float, seed: int = 1, first_index: int = 0, shift_max: float = 0.0):
        """Seeded synthetic particles generated on the device (gen/gen.c's recipe): -> (vols [B,N,N,N] float32,
        truth [B,12] float64 = (R row-major, t))."""
        vols = torch.empty((B, self.N, self.N, self.N), dtype=torch.float32, device=self.device)
        truth = torch.empty((B, 12), dtype=torch.float64, device=self.device)
        self._check(_lib.matcha_synth_particles(self._h, seed, first_index, B, snr, shift_max, _ptr(vols),
                                                _ptr(truth), _stream()))
        return vols, truth

    def set_graphs(self, enable: bool = True):
        """CUDA-graph replay of repeated align_batch calls (needs a non-default current stream)."""
        self._check(_lib.matcha_set_graphs(self._h, 1 if enable else 0))

    def profile_begin(self):
        self._check(_lib.matcha_profile_begin(self._h))

    def profile_end(self):
        """-> {stage: (device ms summed over launches, launches)} since profile_begin (synchronises)."""
        ms = (ctypes.c_double * NUM_STAGES)()
        n = (ctypes.c_int64 * NUM_STAGES)()
        self._check(_lib.matcha_profile_end(self._h, ms, n))
        return {name: (ms[i], n[i]) for i, name in enumerate(STAGES) if n[i] > 0}

    # ---------------------------------------------------------------- stages
    def _vols(self, vols: torch.Tensor, name: str = "vols") -> int:
        if not isinstance(vols, torch.Tensor) or vols.dim() != 4:
            raise ValueError(f"{name} must be a [B, N, N, N] tensor")
        self._arg(vols, name, torch.float32, (vols.shape[0], self.N, self.N, self.N))
        return vols.shape[0]

    def sh_analysis(self, vols: torch.Tensor, shifts: Optional[torch.Tensor] = None, out=None) -> torch.Tensor:
        B = self._vols(vols)
        shape = (B, ncoef(self.L_max), self.R)
        if out is None:
            out = torch.empty(shape, dtype=self.cplx, device=self.device)
        self._arg(out, "out", self.cplx, shape)
        self._arg(shifts, "shifts", self.real, (B, 3), optional=True)
        self._check(_lib.matcha_sh_analysis(self._h, _ptr(vols), B, _ptr(shifts), _ptr(out), _stream()))
        return out

    def corr_coeffs(self, f: torch.Tensor, href: torch.Tensor, L: Optional[int] = None, out=None) -> torch.Tensor:
        L = self.L_max if L is None else L
        B = f.shape[0]
        self._arg(f, "f", self.cplx, (B, ncoef(self.L_max), self.R))
        self._arg(href, "href", self.cplx, (ncoef(self.L_max), self.R))
        if out is None:
            out = torch.empty((B, corr_count(L)), dtype=self.cplx, device=self.device)
        self._arg(out, "out", self.cplx, (B, corr_count(L)))
        self._check(_lib.matcha_corr_coeffs(self._h, _ptr(f), _ptr(href), B, L, _ptr(out), _stream()))
        return out

    def _M(self, M: torch.Tensor, L_M: int) -> int:
        if not isinstance(M, torch.Tensor) or M.dim() != 2:
            raise ValueError("M must be a [B, Mh(L_M)] tensor")
        self._arg(M, "M", self.cplx, (M.shape[0], corr_count(L_M)))
        return M.shape[0]

    def so3_search(self, M: torch.Tensor, L_M: int, L0: int, oversample: int = 2, n_cand: int = 10):
        B = self._M(M, L_M)
        euler = torch.empty((B, n_cand, 3), dtype=self.real, device=self.device)
        score = torch.empty((B, n_cand), dtype=self.real, device=self.device)
        idx = torch.empty((B, n_cand), dtype=torch.int32, device=self.device)
        self._check(_lib.matcha_so3_search(self._h, _ptr(M), L_M, B, L0, oversample, n_cand, _ptr(euler),
                                           _ptr(score), _ptr(idx), _stream()))
        return euler, score, idx

    def eval_corr(self, M: torch.Tensor, L_M: int, L: int, euler: torch.Tensor, derivs: bool = True):
        B = self._M(M, L_M)
        if not isinstance(euler, torch.Tensor) or euler.dim() != 3:
            raise ValueError("euler must be a [B, Q, 3] tensor")
        Q = euler.shape[1]
        self._arg(euler, "euler", self.real, (B, Q, 3))
        val = torch.empty((B, Q), dtype=self.real, device=self.device)
        grad = torch.empty((B, Q, 3), dtype=self.real, device=self.device) if derivs else None
        hess = torch.empty((B, Q, 6), dtype=self.real, device=self.device) if derivs else None
        self._check(_lib.matcha_eval_corr(self._h, _ptr(M), L_M, B, Q, L, _ptr(euler), _ptr(val),
                                          _ptr(grad), _ptr(hess), _stream()))
        return val, grad, hess

    def newton_refine(self, M: torch.Tensor, L_M: int, euler: torch.Tensor, params: Params,
                      grid_idx: Optional[torch.Tensor] = None):
        B = self._M(M, L_M)
        if not isinstance(euler, torch.Tensor) or euler.dim() != 3:
            raise ValueError("euler must be a [B, n_cand, 3] tensor")
        Q = euler.shape[1]
        self._arg(euler, "euler", self.real, (B, Q, 3))
        self._arg(grid_idx, "grid_idx", torch.int32, (B, Q), optional=True)
        euler = euler.clone()
        score = torch.empty((B, Q), dtype=self.real, device=self.device)
        best = torch.empty((B,), dtype=torch.int32, device=self.device)
        p = params.c()
        self._check(_lib.matcha_newton_refine(self._h, _ptr(M), L_M, B, Q, ctypes.byref(p), _ptr(euler),
                                              _ptr(grid_idx), _ptr(score), _ptr(best), _stream()))
        return euler, score, best

    def translation_update(self, vols: torch.Tensor, ref: torch.Tensor, euler: torch.Tensor, window: int,
                           upsample: int = 0):
        B = self._vols(vols)
        self._arg(ref, "ref", torch.float32, (self.N, self.N, self.N))
        self._arg(euler, "euler", self.real, (B, 3))
        shifts = torch.empty((B, 3), dtype=self.real, device=self.device)
        peak = torch.empty((B,), dtype=self.real, device=self.device)
        self._check(_lib.matcha_translation_update(self._h, _ptr(vols), B, _ptr(ref), _ptr(euler),
                                                   window, upsample, _ptr(shifts), _ptr(peak), _stream()))
        return shifts, peak

    def align_batch(self, vols: torch.Tensor, ref: Optional[torch.Tensor], params: Params,
                    ref_coeffs: Optional[torch.Tensor] = None, out=None) -> torch.Tensor:
        """poses [B, 8] = (alpha, beta, gamma, t_x, t_y, t_z, score, best_cand)."""
        B = self._vols(vols)
        self._arg(ref, "ref", torch.float32, (self.N, self.N, self.N), optional=True)
        self._arg(ref_coeffs, "ref_coeffs", self.cplx, (ncoef(self.L_max), self.R), optional=True)
        if out is None:
            out = torch.empty((B, 8), dtype=self.real, device=self.device)
        self._arg(out, "out", self.real, (B, 8))
        p = params.c()
        self._check(_lib.matcha_align_batch(self._h, _ptr(vols), B, _ptr(ref), _ptr(ref_coeffs), ctypes.byref(p),
                                            _ptr(out), _stream()))
        return out

    # ---------------------------------------------------------------- ball-harmonic radial basis
    def ball_kmax(self, lam: float = 0.0):
        """-> (Kmax, [|K_l| for l = 0..L_max]) of the ball basis with cutoff lam (<= 0: pi (R - 1/2))."""
        K = (ctypes.c_int32 * (self.L_max + 1))()
        km = int(_lib.matcha_ball_kmax(self._h, lam, K))
        if km < 0:
            self._check(-1)
        return km, list(K)

    def ball_transform(self, F: torch.Tensor, lam: float = 0.0, out=None) -> torch.Tensor:
        """Shell coefficients [B, ncoef, R] -> ball coefficients [B, ncoef, Kmax] (App. A.1)."""
        B = F.shape[0]
        self._arg(F, "F", self.cplx, (B, ncoef(self.L_max), self.R))
        km, _ = self.ball_kmax(lam)
        if out is None:
            out = torch.empty((B, ncoef(self.L_max), km), dtype=self.cplx, device=self.device)
        self._arg(out, "out", self.cplx, (B, ncoef(self.L_max), km))
        self._check(_lib.matcha_ball_transform(self._h, _ptr(F), B, lam, _ptr(out), _stream()))
        return out

    def corr_coeffs_ball(self, fb: torch.Tensor, hb: torch.Tensor, L: Optional[int] = None, lam: float = 0.0,
                         out=None) -> torch.Tensor:
        """M^l_mn = sum_{k in K_l} f^_klm conj(h^_kln) -> [B, Mh(L)] half plane (rank <= |K_l|)."""
        L = self.L_max if L is None else L
        km, _ = self.ball_kmax(lam)
        B = fb.shape[0]
        self._arg(fb, "fb", self.cplx, (B, ncoef(self.L_max), km))
        self._arg(hb, "hb", self.cplx, (ncoef(self.L_max), km))
        if out is None:
            out = torch.empty((B, corr_count(L)), dtype=self.cplx, device=self.device)
        self._arg(out, "out", self.cplx, (B, corr_count(L)))
        self._check(_lib.matcha_corr_coeffs_ball(self._h, _ptr(fb), _ptr(hb), B, L, lam, _ptr(out), _stream()))
        return out

    def align_multi(self, vols: torch.Tensor, refs: Optional[torch.Tensor], params: Params,
                    ref_coeffs: Optional[torch.Tensor] = None, out=None) -> torch.Tensor:
        """Multi-template alignment: refs [T, N, N, N] -> poses [B, 9] (..., template index)."""
        B = self._vols(vols)
        nt = refs.shape[0] if refs is not None else ref_coeffs.shape[0]
        self._arg(refs, "refs", torch.float32, (nt, self.N, self.N, self.N), optional=True)
        self._arg(ref_coeffs, "ref_coeffs", self.cplx, (nt, ncoef(self.L_max), self.R), optional=True)
        if out is None:
            out = torch.empty((B, 9), dtype=self.real, device=self.device)
        self._arg(out, "out", self.real, (B, 9))
        p = params.c()
        self._check(_lib.matcha_align_multi(self._h, _ptr(vols), B, _ptr(refs), nt, _ptr(ref_coeffs), ctypes.byref(p),
                                            _ptr(out), _stream()))
        return out

    def reconstruct(self, vols: torch.Tensor, poses: torch.Tensor, n_classes: int = 1, class_col: int = -1,
                    first_index: int = 0):
        """Half-map sums of the aligned particles: -> (sums [n_classes, 2, N, N, N] real,
        counts [n_classes, 2] int32).  poses [B, stride]: columns 0..5 = (alpha, beta, gamma, tx, ty, tz)."""
        B = self._vols(vols)
        if not isinstance(poses, torch.Tensor) or poses.dim() != 2:
            raise ValueError("poses must be a [B, stride] tensor")
        self._arg(poses, "poses", self.real, (B, poses.shape[1]))
        sums = torch.empty((n_classes, 2, self.N, self.N, self.N), dtype=self.real, device=self.device)
        counts = torch.empty((n_classes, 2), dtype=torch.int32, device=self.device)
        self._check(_lib.matcha_reconstruct(self._h, _ptr(vols), B, _ptr(poses), poses.shape[1], class_col, n_classes,
                                            first_index, _ptr(sums), _ptr(counts), _stream()))
        return sums, counts

    def align_batch_host(self, vols_host: torch.Tensor, ref_host: torch.Tensor, params: Params,
                         out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """End-to-end on host (ideally pinned) buffers: H2D chunks overlapped with compute; syncs."""
        n3 = (self.N,) * 3

        def host(t, name, dtype, shape):
            if not isinstance(t, torch.Tensor) or t.is_cuda or not t.is_contiguous() or t.dtype != dtype:
                raise TypeError(f"{name} must be a contiguous host {dtype} tensor")
            if tuple(t.shape) != tuple(shape):
                raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")

        B = vols_host.shape[0]
        host(vols_host, "vols_host", torch.float32, (B,) + n3)
        host(ref_host, "ref_host", torch.float32, n3)
        if out is None:
            out = torch.empty((B, 8), dtype=self.real, pin_memory=True)
        host(out, "out", self.real, (B, 8))
        p = params.c()
        self._check(_lib.matcha_align_batch_host(self._h, ctypes.c_void_p(vols_host.data_ptr()), B,
                                                 ctypes.c_void_p(ref_host.data_ptr()), ctypes.byref(p),
                                                 ctypes.c_void_p(out.data_ptr()), _stream()))
        return out
