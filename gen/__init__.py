"""Seeded synthetic-input generator (test/bench infrastructure, not the method).

Wraps ``gen/libmatcha_gen.so`` (plain C, ``gen/gen.c``).  It holds none of the
method's arithmetic: it draws Philox4x32-10 random numbers and renders the
Gaussian-blob phantom of DESIGN.md "Input recipe".  Both the FP64 oracle and the
CUDA path consume the float32 volumes produced here, so their inputs are
bit-identical.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

REF_SEED = 0x5EED  # reference blobs keyed (0x5EED, 0)
N_BLOBS = 32


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libmatcha_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)} gen`")
        lib = ctypes.CDLL(path)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        lib.gen_reference_blobs.argtypes = [ctypes.c_uint64, ctypes.c_int, dp]
        lib.gen_render.argtypes = [dp, ctypes.c_int, ctypes.c_int, dp, dp, fp]
        lib.gen_render.restype = ctypes.c_double
        lib.gen_particle_pose.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double, dp, dp, dp]
        lib.gen_particles.argtypes = [ctypes.c_uint64, dp, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                      ctypes.c_double, dp, fp, dp, ctypes.c_int]
        lib.gen_particles.restype = ctypes.c_double
        _LIB = lib
    return _LIB


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) if a is not None else None


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def reference_blobs(seed: int = REF_SEED, nblobs: int = N_BLOBS) -> np.ndarray:
    b = np.zeros((nblobs, 10), np.float64)
    _lib().gen_reference_blobs(seed, nblobs, _dp(b))
    return b


def render(blobs: np.ndarray, N: int, R=None, t=None):
    """f(x) = h(R^T (x - c - t)/(N/2)); returns (volume float32 [N,N,N] z-major, mean square)."""
    vol = np.zeros((N, N, N), np.float32)
    Rm = None if R is None else np.ascontiguousarray(R, np.float64).reshape(9)
    tv = None if t is None else np.ascontiguousarray(t, np.float64).reshape(3)
    ms = _lib().gen_render(_dp(np.ascontiguousarray(blobs)), blobs.shape[0], N, _dp(Rm), _dp(tv), _fp(vol))
    return vol, ms


SHIFT_ZERO, SHIFT_UNIFORM, SHIFT_FIXED = 0, 1, 2


@dataclass
class Batch:
    vols: np.ndarray      # float32 [B,N,N,N]
    ref: np.ndarray       # float32 [N,N,N]
    truth_R: np.ndarray   # float64 [B,3,3]  planted g*
    truth_t: np.ndarray   # float64 [B,3]    planted t* (x,y,z voxels, particle frame)
    sigma: float
    p_ref: float


def particles(N: int, B: int, snr: float, seed: int = 1, first: int = 0, shift_mode: int = SHIFT_ZERO,
              shift_max: float = 0.0, fixed_shift=(0.0, 0.0, 0.0), nthreads: int | None = None,
              out: np.ndarray | None = None) -> Batch:
    """Particles first..first+B-1: f_p = S_{t_p}(g_p o h) + eta_p (SURVEY 8(d) recipe)."""
    blobs = reference_blobs()
    ref, p_ref = render(blobs, N)
    vols = out if out is not None else np.empty((B, N, N, N), np.float32)
    assert vols.dtype == np.float32 and vols.flags.c_contiguous and vols.shape == (B, N, N, N)
    truth = np.zeros((B, 12), np.float64)
    fs = np.ascontiguousarray(fixed_shift, np.float64)
    nt = nthreads or max(1, min(64, os.cpu_count() or 1))
    snr_c = float(snr) if (snr is not None and np.isfinite(snr)) else -1.0
    sigma = _lib().gen_particles(seed, _dp(blobs), blobs.shape[0], N, first, B, snr_c, p_ref, shift_mode,
                                 shift_max, _dp(fs), _fp(vols), _dp(truth), nt)
    return Batch(vols, ref, truth[:, :9].reshape(B, 3, 3).copy(), truth[:, 9:].copy(), sigma, p_ref)
