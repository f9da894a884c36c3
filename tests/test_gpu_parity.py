"""GPU parity: the CUDA path through the C ABI vs the FP64 oracle, element by element on the same seeded
inputs (tolerances: SURVEY.md 8(c) / tests/parity_util.py).  Run on a B200 with `pytest -m gpu`."""
import numpy as np
import pytest
import torch

import gen
import oracle as O
from parity_util import (TOL_ROT_DEG, c_tol, g_tol, h_tol, rot_err_deg, topk_index_must_match)

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2603_15285_b200 as mt  # noqa: E402  (raises if libmatcha.so is missing: no CPU fallback)

DEV = torch.device("cuda", 0)
rng = np.random.default_rng(7)


def cuda(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def to_np(t):
    return t.detach().cpu().numpy()


@pytest.fixture(scope="module", params=["fp32", "fp64"])
def prec(request):
    return request.param


def handle(N, L, prec="fp32", max_batch=64):
    return mt.Handle(N=N, L_max=L, quad_oversample=2, max_batch=max_batch, precision=prec)


# ------------------------------------------------------------------ stage 1
@pytest.mark.parametrize("N,L,B", [(32, 8, 5), (64, 32, 3), (16, 5, 7), (128, 64, 2)])
def test_sh_analysis_parity(N, L, B, prec):
    b = gen.particles(N, B, 0.1, seed=21, shift_mode=gen.SHIFT_UNIFORM, shift_max=2.0)
    h = handle(N, L, prec)
    vols = cuda(b.vols)
    shifts = rng.uniform(-3, 3, size=(B, 3))
    shifts[0] = [N / 2, -N / 2 + 1, 0.5]  # samples leave the box: zero extension (reading C5)
    for sh in (None, shifts):
        F = to_np(h.sh_analysis(vols, None if sh is None else cuda(sh, h.real)))
        Fo = O.sh_analysis_batch(b.vols, L, 2, sh)
        for p in range(B):
            scale = np.abs(Fo[p]).max()
            tol = (1e-11 if prec == "fp64" else 2e-5) * scale
            assert np.abs(F[p] - Fo[p]).max() <= tol, (p, np.abs(F[p] - Fo[p]).max() / scale)


@pytest.mark.parametrize("N,L,B", [(64, 32, 150), (32, 8, 160), (16, 5, 48), (48, 20, 40), (96, 48, 40),
                                   (64, 60, 40), (128, 64, 40)])
def test_sh_analysis_tensor_core_path_parity(N, L, B):
    """Batches of at least a quarter of the SMs take the persistent tensor-core ring kernel (fp16 hi/lo split DFT,
    z-sorted rings, plane ring buffer) -- compared with the oracle on sampled particles, unshifted and shifted
    (including shifts that push samples out of the box and planes outside the volume), at the bench's launch
    configuration (sub-batches of whole waves of particles).  L = 48 and 60 take the two-k-round variant (32 rings
    per tile, Kh <= 64: c3's stage 1 on tensor cores); 128^3 / L = 64 (c5) the 16-ring, 2-plane-slot
    variant whose m = 64 rows come from the samplers (2(L+1) = 130 > 128 MMA rows)."""
    b = gen.particles(N, B, 0.1, seed=26)
    h = handle(N, L, "fp32", max_batch=B)
    vols = cuda(b.vols)
    shifts = rng.uniform(-3, 3, size=(B, 3))
    shifts[1] = [N / 2, -N / 2 + 1, 0.5]
    shifts[B - 1] = [0.25, -0.75, -N / 2 - 0.5]
    sample = [0, 1, B // 2, B - 1]
    for sh in (None, shifts):
        F = to_np(h.sh_analysis(vols, None if sh is None else cuda(sh, h.real)))
        for p in sample:
            Fo = O.sh_analysis(b.vols[p], L, 2, None if sh is None else sh[p])
            scale = np.abs(Fo).max()
            assert np.abs(F[p] - Fo).max() <= 2e-5 * scale, (p, np.abs(F[p] - Fo).max() / scale)


def test_sh_analysis_empty_batch():
    h = handle(16, 4)
    out = h.sh_analysis(torch.empty((0, 16, 16, 16), device=DEV))
    assert out.shape[0] == 0


# ------------------------------------------------------------------ stage 2
@pytest.mark.parametrize("N,L,Lc", [(64, 32, 32), (64, 32, 16), (32, 8, 8)])
def test_corr_coeffs_parity(N, L, Lc, prec):
    b = gen.particles(N, 3, 0.1, seed=22)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    h = handle(N, L, prec)
    M = to_np(h.corr_coeffs(cuda(Fo, h.cplx), cuda(Ho, h.cplx), Lc))
    for p in range(3):
        Mo = O.full_to_half(O.corr_full(Fo[p], Ho, Lc), Lc)
        scale = np.abs(Mo).max()
        assert np.abs(M[p] - Mo).max() <= (1e-12 if prec == "fp64" else 1e-5) * scale


@pytest.mark.parametrize("L,R,B,Lc", [(48, 48, 70, 48), (64, 64, 9, 61), (100, 100, 3, 100), (20, 20, 37, 20),
                                      (7, 4, 300, 7)])
def test_corr_coeffs_tiled_parity(L, R, B, Lc, prec):
    """Stage 2 on the tiled SIMT kernel (every degree / shell count the tensor-core kernel does not take, and FP64):
    row tiles spanning particles with ragged tails, column tiles of 2l+1 > 64, shell chunks with R % 16 != 0 (R = N/2, N a multiple of 8).
    F and H are seeded complex Gaussians shaped like shell coefficients (inputs, not method output)."""
    r = np.random.default_rng(L * 1000 + R)
    nc = mt.ncoef(L)
    scale = (1.0 / (1.0 + np.arange(nc)))[:, None] * np.ones((1, R))
    F = (r.normal(size=(B, nc, R)) + 1j * r.normal(size=(B, nc, R))) * scale
    H = (r.normal(size=(nc, R)) + 1j * r.normal(size=(nc, R))) * scale
    for l in range(L + 1):  # m = 0 entries real (reading C3)
        F[:, l * (l + 1) // 2, :] = F[:, l * (l + 1) // 2, :].real
        H[l * (l + 1) // 2, :] = H[l * (l + 1) // 2, :].real
    h = handle(2 * R, L, prec)
    M = to_np(h.corr_coeffs(cuda(F, h.cplx), cuda(H, h.cplx), Lc))
    Fq = to_np(cuda(F, h.cplx)).astype(np.complex128)
    Hq = to_np(cuda(H, h.cplx)).astype(np.complex128)
    for p in sorted({0, B // 2, B - 1}):
        Mo = O.full_to_half(O.corr_full(Fq[p], Hq, Lc), Lc)
        assert np.abs(M[p] - Mo).max() <= (1e-12 if prec == "fp64" else 1e-5) * np.abs(Mo).max(), p


# ------------------------------------------------------------------ C_L, grad, Hess (the evaluation kernel)
@pytest.mark.parametrize("N,L,Leval", [(64, 32, 32), (64, 32, 24), (64, 32, 8), (32, 8, 8), (128, 64, 64),
                                       (64, 100, 100), (64, 100, 60)])
def test_eval_corr_parity(N, L, Leval, prec):
    b = gen.particles(N, 2, 0.1, seed=23)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    Q = 12
    eul = np.stack([rng.uniform(0, 2 * np.pi, (2, Q)), rng.uniform(0, np.pi, (2, Q)),
                    rng.uniform(0, 2 * np.pi, (2, Q))], -1)
    eul[:, 0, 1] = 0.02          # near the poles (reading C16 clamp never triggers here)
    eul[:, 1, 1] = np.pi - 0.03
    eul[:, 2, 1] = np.pi / 2
    h = handle(N, L, prec)
    Mh = np.stack([O.full_to_half(O.corr_full(Fo[p], Ho, L), L) for p in range(2)])
    val, grad, hess = h.eval_corr(cuda(Mh, h.cplx), L, Leval, cuda(eul, h.real))
    val, grad, hess = to_np(val), to_np(grad), to_np(hess)
    eul_used = to_np(cuda(eul, h.real)).astype(np.float64)  # the rotations the GPU actually saw
    fp64 = prec == "fp64"
    for p in range(2):
        Mf = O.corr_full(Fo[p], Ho, Leval)
        E = O.energy(Fo[p], Ho, Leval)
        for q in range(Q):
            C, g, H = O.eval_corr(Mf, Leval, eul_used[p, q])
            assert abs(val[p, q] - C) <= c_tol(C, E, fp64), (p, q, val[p, q], C)
            assert np.abs(grad[p, q] - g).max() <= g_tol(g, E, Leval, fp64), (p, q)
            assert np.abs(hess[p, q] - H).max() <= h_tol(H, E, Leval, fp64), (p, q, hess[p, q], H)


@pytest.mark.parametrize("Q", [1, 2, 3, 4, 5, 9, 10])
@pytest.mark.parametrize("derivs", [True, False], ids=["derivs", "value"])
def test_eval_corr_candidate_groups(Q, derivs, prec):
    """Every register-group size the kernel picks for Q candidates (pick_cg: 1, 2, 4, 5 in FP32; 1, 2 in FP64),
    with and without derivatives (the value-only path is the final C_{L_J} of newton_refine)."""
    N, L = 64, 32
    b = gen.particles(N, 1, 0.1, seed=29)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    r = np.random.default_rng(Q)
    eul = np.stack([r.uniform(0, 2 * np.pi, (1, Q)), r.uniform(0, np.pi, (1, Q)), r.uniform(0, 2 * np.pi, (1, Q))], -1)
    h = handle(N, L, prec)
    Mf = O.corr_full(Fo[0], Ho, L)
    val, grad, hess = h.eval_corr(cuda(O.full_to_half(Mf, L)[None], h.cplx), L, L, cuda(eul, h.real), derivs)
    eul_used = to_np(cuda(eul, h.real)).astype(np.float64)
    E = O.energy(Fo[0], Ho, L)
    fp64 = prec == "fp64"
    val = to_np(val)
    for q in range(Q):
        C, g, H = O.eval_corr(Mf, L, eul_used[0, q])
        assert abs(val[0, q] - C) <= c_tol(C, E, fp64), (q, val[0, q], C)
        if derivs:
            assert np.abs(to_np(grad)[0, q] - g).max() <= g_tol(g, E, L, fp64), q
            assert np.abs(to_np(hess)[0, q] - H).max() <= h_tol(H, E, L, fp64), q


# ------------------------------------------------------------------ stage 3
@pytest.mark.parametrize("N,L,L0,K,nc", [(64, 32, 8, 2, 10), (32, 8, 4, 2, 4), (128, 64, 12, 2, 16),
                                         (32, 8, 8, 1, 32), (64, 32, 30, 2, 10)])
def test_so3_search_parity(N, L, L0, K, nc, prec):
    B = 3
    b = gen.particles(N, B, 0.1, seed=24)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    h = handle(N, L, prec)
    Mh = np.stack([O.full_to_half(O.corr_full(Fo[p], Ho, L), L) for p in range(B)])
    eul, sc, idx = h.so3_search(cuda(Mh, h.cplx), L, L0, K, nc)
    eul, sc, idx = to_np(eul), to_np(sc), to_np(idx)
    compared = 0
    for p in range(B):
        Mf = O.corr_full(Fo[p], Ho, L0)
        grid = O.grid_eval(Mf, L0, K)
        all_idx, all_sc, n = O.find_maxima(grid, 100000)
        all_idx, all_sc = all_idx[:n], all_sc[:n]
        E0 = O.energy(Fo[p], Ho, L0)
        for k in range(nc):
            if k >= n:
                assert idx[p, k] == -1 and np.isneginf(sc[p, k])
                continue
            if topk_index_must_match(all_sc, all_idx, k, grid, E0):
                compared += 1
                assert idx[p, k] == all_idx[k], (p, k)
                assert abs(sc[p, k] - all_sc[k]) <= c_tol(all_sc[k], E0, prec == "fp64")
                assert np.allclose(eul[p, k], O.grid_node_euler(all_idx[k], L0, K), atol=1e-6)
    assert compared >= B * min(nc, 3)


# ------------------------------------------------------------------ stage 4
def _oracle_stable(Mf, bands, iters, eul0, idx0, e_ref, seed):
    """Candidates whose oracle trajectory is insensitive to an FP32-sized perturbation (1e-6 relative on M,
    start angles rounded to float32).  Weak candidates on a noisy landscape take huge, chaotic Newton steps
    (SURVEY 8(c) "parity unpinned: noisy-landscape Newton paths"): there several results are correct, so
    only their validity is checked."""
    r = np.random.default_rng(seed)
    Mp = Mf * (1 + 1e-6 * r.normal(size=Mf.shape))
    ep, _, _ = O.refine(Mp, bands, iters, eul0.astype(np.float32).astype(np.float64), idx0)
    return np.array([rot_err_deg(ep[c], e_ref[c]) < 0.01 for c in range(len(e_ref))])


@pytest.mark.parametrize("N,L,bands,nc,iters", [(64, 32, [8, 12, 16, 24, 32], 10, 1), (32, 8, [4, 6, 8], 4, 2),
                                                (64, 32, [16, 32], 5, 3)])
def test_newton_refine_parity(N, L, bands, nc, iters, prec):
    B = 4
    b = gen.particles(N, B, 0.1, seed=25)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    L0, K = bands[0], 2
    h = handle(N, L, prec)
    eul0 = np.zeros((B, nc, 3))
    idx0 = np.zeros((B, nc), np.int64)
    Mh = []
    for p in range(B):
        Mf = O.corr_full(Fo[p], Ho, L)
        Mh.append(O.full_to_half(Mf, L))
        idx, sc, n = O.find_maxima(O.grid_eval(O.corr_full(Fo[p], Ho, L0), L0, K), nc)
        idx0[p] = idx
        eul0[p] = [O.grid_node_euler(i, L0, K) if i >= 0 else np.zeros(3) for i in idx]
    params = mt.Params(bands=bands, newton_iters=iters, n_cand=nc, oversample=K)
    eg, sg, bg = h.newton_refine(cuda(np.stack(Mh), h.cplx), L, cuda(eul0, h.real), params,
                                 cuda(idx0.astype(np.int32)))
    eg, sg, bg = to_np(eg), to_np(sg), to_np(bg)
    nbad = ntot = 0
    for p in range(B):
        Mf = O.corr_full(Fo[p], Ho, L)
        eo, so, bo = O.refine(Mf, bands, iters, eul0[p], idx0[p])
        stable = _oracle_stable(Mf, bands, iters, eul0[p], idx0[p], eo, seed=p)
        E = O.energy(Fo[p], Ho, bands[-1])
        for c in range(nc):
            if idx0[p, c] < 0:
                assert np.isneginf(sg[p, c])
                continue
            # every candidate: valid chart point with a finite score
            assert np.isfinite(sg[p, c]) and 0 <= eg[p, c, 1] <= np.pi + 1e-6
            assert 0 <= eg[p, c, 0] < 2 * np.pi + 1e-6 and 0 <= eg[p, c, 2] < 2 * np.pi + 1e-6
            if not stable[c]:
                continue
            ntot += 1
            err = rot_err_deg(eg[p, c], eo[c])
            if err > TOL_ROT_DEG:
                nbad += 1
            else:
                assert abs(sg[p, c] - so[c]) <= c_tol(so[c], E, prec == "fp64")
        # the selected pose: same candidate, or (reading C23, several correct results) another pose that the oracle
        # itself scores at least as high as its own choice -- e.g. a chaotic candidate whose FP32 path climbed to a
        # better maximum than its FP64 path; the GPU's reported score must be the oracle's score at that pose
        assert stable[bo]
        if bg[p] != bo and rot_err_deg(eg[p, bg[p]], eo[bo]) > TOL_ROT_DEG:
            Cg = O.eval_corr(Mf, bands[-1], eg[p, bg[p]].astype(np.float64))[0]
            assert abs(sg[p, bg[p]] - Cg) <= c_tol(Cg, E, prec == "fp64"), (p, sg[p, bg[p]], Cg)
            assert Cg >= so[bo] - c_tol(so[bo], E), (p, bg[p], bo, Cg, so[bo])
    assert ntot >= B and nbad <= 0.001 * ntot, (nbad, ntot)


# ------------------------------------------------------------------ whole path
def _align_compare(N, L, bands, nc, snr, B, sample, prec="fp32", max_batch=64, seed=31, L0=None):
    b = gen.particles(N, B, snr, seed=seed)
    h = handle(N, L, prec, max_batch=max_batch)
    params = mt.Params(bands=bands, n_cand=nc, oversample=2)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    P = dict(L=L, qover=2, L0=bands[0], K=2, ncand=nc, bands=bands, iters=1, T=1, W=0)
    sel = np.arange(B) if sample is None else np.unique(np.linspace(0, B - 1, sample).astype(int))
    po = O.align_batch(b.vols[sel], b.ref, P)
    Ho = O.sh_analysis(b.ref, L)
    bad = []
    for i, p in enumerate(sel):
        err = rot_err_deg(poses[p, :3], po[i, :3])
        if err > TOL_ROT_DEG:
            # several results can be correct (C23): accept a different candidate whose oracle score ties
            Fo = O.sh_analysis(b.vols[p], L)
            Mf = O.corr_full(Fo, Ho, L)
            C_g = O.eval_corr(Mf, L, poses[p, :3])[0]
            E = O.energy(Fo, Ho, L)
            if abs(C_g - po[i, 6]) > c_tol(po[i, 6], E):
                bad.append((p, err))
    return bad, len(sel), poses, b


def test_align_c1_noise_free_exact():
    """c1 rotation part (32^3, L0=4 -> 8, N_C=4, noise-free): GPU == oracle, both near the planted truth."""
    bad, n, poses, b = _align_compare(32, 8, [4, 6, 8], 4, float("inf"), 8, None)
    assert not bad
    for p in range(8):
        assert O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) < 0.1


def test_align_parity_1000_particles_c1_shape_noisy():
    """>= 1,000 compared particles (SURVEY 8(c) pass rate >= 99.9%) at the c1 shape with SNR 0.1."""
    bad, n, _, _ = _align_compare(32, 8, [4, 6, 8], 4, 0.1, 1000, None, max_batch=256, seed=32)
    assert len(bad) <= 1, bad


def test_align_parity_c2_full_size_sampled():
    """c2 at full size (1,000 x 64^3, L0=8 -> 32, N_C=10) in the bench's launch configuration; the oracle
    recomputes a sample of particles one by one."""
    bad, n, poses, b = _align_compare(64, 32, [8, 12, 16, 24, 32], 10, 0.1, 1000, 24, max_batch=1000, seed=33)
    assert not bad, bad
    errs = [O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) for p in range(0, 1000, 50)]
    assert np.median(errs) < 1.0  # sanity vs planted truth (median ~0.3 deg at SNR 0.1)


def test_align_ragged_chunks_and_fp64():
    bad, n, _, _ = _align_compare(32, 8, [4, 6, 8], 4, 0.1, 37, None, prec="fp64", max_batch=16, seed=34)
    assert not bad


def test_align_bitwise_deterministic():
    b = gen.particles(32, 20, 0.1, seed=35)
    h = handle(32, 8)
    params = mt.Params(bands=[4, 6, 8], n_cand=4)
    p1 = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    p2 = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    assert np.array_equal(p1, p2)
    # shard invariance: particles 7..19 alone give the same bits (multi-GPU invariant)
    p3 = to_np(h.align_batch(cuda(b.vols[7:]), cuda(b.ref), params))
    assert np.array_equal(p1[7:], p3)


def test_align_host_path_matches_device_path():
    b = gen.particles(32, 40, 0.1, seed=36)
    h = handle(32, 8, max_batch=16)
    params = mt.Params(bands=[4, 6, 8], n_cand=4)
    pd = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    ph = h.align_batch_host(torch.from_numpy(b.vols).pin_memory(), torch.from_numpy(b.ref).pin_memory(), params)
    assert np.array_equal(pd, ph.numpy())


def test_invalid_arguments_rejected():
    h = handle(32, 8)
    M = torch.zeros((1, mt.corr_count(8)), dtype=torch.complex64, device=DEV)
    with pytest.raises(mt.MatchaError):
        h.so3_search(M, 8, 9)  # L0 > L_M
    with pytest.raises(mt.MatchaError):
        h.newton_refine(M, 8, torch.zeros((1, 4, 3), device=DEV), mt.Params(bands=[6, 4]))
    with pytest.raises(mt.MatchaError):
        mt.Handle(N=33, L_max=8)


# ------------------------------------------------------------------ stage 5: translation (App. C)
@pytest.mark.parametrize("N,W,shift_mode", [(32, 4, gen.SHIFT_FIXED), (32, 3, gen.SHIFT_UNIFORM), (64, 8, gen.SHIFT_UNIFORM),
                                            (32, 8, gen.SHIFT_UNIFORM), (24, 6, gen.SHIFT_FIXED),
                                            (40, 4, gen.SHIFT_UNIFORM), (56, 5, gen.SHIFT_FIXED)])
def test_translation_update_parity(N, W, shift_mode, prec):
    B = 4
    b = gen.particles(N, B, 1.0, seed=41, shift_mode=shift_mode, shift_max=W - 1.0, fixed_shift=(1.0, -2.0, 1.0))
    eul = np.array([O.matrix_to_euler(R) for R in b.truth_R])
    eul[1] += 0.01  # a slightly wrong rotation: the peak is still well defined
    h = handle(N, 8, prec)
    sh, pk = h.translation_update(cuda(b.vols), cuda(b.ref), cuda(eul, h.real), W)
    sh, pk = to_np(sh), to_np(pk)
    eul_used = to_np(cuda(eul, h.real)).astype(np.float64)
    for p in range(B):
        so, po = O.translation(b.vols[p], b.ref, eul_used[p], W)
        assert np.abs(sh[p] - so).max() < (1e-6 if prec == "fp64" else 2e-3), (p, sh[p], so)
        assert abs(pk[p] - po) <= (1e-9 if prec == "fp64" else 1e-4) * abs(po)
        assert np.abs(sh[p] - b.truth_t[p]).max() < 0.6  # near the planted shift


def test_translation_c3_shape_vs_oracle_and_truth():
    """c3's 96^3 / W = 6 at SNR 0.05 on a batch that spans several CTAs, at the TRUE rotations (FP32 angles, the
    handle's precision): the shifts recover the planted U[-4,4]^3 shifts (< 0.6 voxel), and 2 particles are
    compared with the oracle's direct windowed correlation (App. C; reading C18).  (Round 1 fed float64
    angles to the FP32 handle here; the binding now rejects that, see test_binding_rejects_wrong_dtypes.)"""
    N, W, B = 96, 6, 6
    b = gen.particles(N, B, 0.05, seed=43, shift_mode=gen.SHIFT_UNIFORM, shift_max=4.0)
    h = handle(N, 8)
    eul = np.array([O.matrix_to_euler(R) for R in b.truth_R])
    sh, pk = h.translation_update(cuda(b.vols), cuda(b.ref), cuda(eul, h.real), W)
    sh, pk = to_np(sh), to_np(pk)
    assert np.abs(sh - b.truth_t).max() < 0.6, np.abs(sh - b.truth_t).max()
    eul_used = to_np(cuda(eul, h.real)).astype(np.float64)
    for p in (0, 4):
        so, po = O.translation(b.vols[p], b.ref, eul_used[p], W)
        assert np.abs(sh[p] - so).max() < 2e-3, (p, sh[p], so)
        assert abs(pk[p] - po) <= 1e-4 * abs(po)


def test_binding_rejects_wrong_dtypes():
    """Tensors cross the C ABI as raw pointers: the binding must refuse a float64 tensor handed to an FP32 handle
    (and wrong shapes / devices / int64 indices) instead of letting the kernel reinterpret its bytes."""
    N = 32
    h = handle(N, 8)
    vols = torch.zeros((2, N, N, N), device=DEV)
    ref = torch.zeros((N, N, N), device=DEV)
    with pytest.raises(TypeError):
        h.translation_update(vols, ref, torch.zeros((2, 3), dtype=torch.float64, device=DEV), 4)
    with pytest.raises(ValueError):
        h.translation_update(vols, ref, torch.zeros((2, 4), device=DEV), 4)
    with pytest.raises(ValueError):
        h.translation_update(vols, ref.cpu(), torch.zeros((2, 3), device=DEV), 4)
    M = torch.zeros((2, mt.corr_count(8)), dtype=torch.complex64, device=DEV)
    with pytest.raises(TypeError):
        h.eval_corr(M, 8, 8, torch.zeros((2, 3, 3), dtype=torch.float64, device=DEV))
    with pytest.raises(TypeError):
        h.newton_refine(M, 8, torch.zeros((2, 4, 3), device=DEV), mt.Params(bands=[4, 8], n_cand=4),
                        grid_idx=torch.zeros((2, 4), dtype=torch.int64, device=DEV))
    with pytest.raises(TypeError):
        h.eval_corr(M.to(torch.complex128), 8, 8, torch.zeros((2, 3, 3), device=DEV))
    with pytest.raises(TypeError):
        h.align_batch(vols.double(), ref, mt.Params(bands=[4, 8], n_cand=4))
    with pytest.raises(TypeError):
        h.align_batch(vols, ref, mt.Params(bands=[4, 8], n_cand=4),
                      ref_coeffs=torch.zeros((mt.ncoef(8), N // 2), dtype=torch.complex128, device=DEV))
    with pytest.raises(TypeError):
        h.sh_analysis(vols, torch.zeros((2, 3), dtype=torch.float64, device=DEV))
    h64 = handle(N, 8, "fp64")
    with pytest.raises(TypeError):
        h64.translation_update(vols, ref, torch.zeros((2, 3), dtype=torch.float32, device=DEV), 4)
    with pytest.raises(mt.MatchaError):  # W > N/4 (SPEC WindowTooLarge)
        h.align_batch_host(torch.zeros((2, N, N, N)), torch.zeros((N, N, N)),
                           mt.Params(bands=[4, 8], n_cand=4, n_alternations=2, shift_window=N // 4 + 1))


def test_translation_integer_shifts_exact_gpu():
    N = 32
    ref = gen.render(gen.reference_blobs(), N)[0]
    shifts = [(0, 0, 0), (3, -2, 1), (-4, 4, -1), (1, 1, -3)]
    vols = np.stack([np.roll(ref, shift=(t[2], t[1], t[0]), axis=(0, 1, 2)) for t in shifts])
    h = handle(N, 8, "fp64")
    sh, _ = h.translation_update(cuda(vols), cuda(ref), cuda(np.zeros((4, 3)), h.real), 4)
    assert np.abs(to_np(sh) - np.array(shifts, float)).max() < 1e-9


def test_alternation_c1_exact_recovery():
    """configs[0]: one noise-free 32^3 volume, known rotation + integer shift (1,-2,1), L0=4 -> 8, N_C=4, T=8."""
    b = gen.particles(32, 2, float("inf"), seed=12, shift_mode=gen.SHIFT_FIXED, fixed_shift=(1.0, -2.0, 1.0))
    h = handle(32, 8)
    params = mt.Params(bands=[4, 6, 8], n_cand=4, oversample=2, n_alternations=8, shift_window=4)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    po = O.align_batch(b.vols, b.ref, dict(L=8, qover=2, L0=4, K=2, ncand=4, bands=[4, 6, 8], iters=1, T=8, W=4))
    for p in range(2):
        assert rot_err_deg(poses[p, :3], po[p, :3]) < TOL_ROT_DEG
        assert np.abs(poses[p, 3:6] - po[p, 3:6]).max() < 0.1
        assert O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) < 0.05
        assert np.abs(poses[p, 3:6] - b.truth_t[p]).max() < 0.01


def test_alternation_c3_shape_sampled():
    """configs[2] shape: 96^3, SNR 0.05, L0=8 -> 48, shifts U[-4,4]^3, T=3, W=6 (App. C); oracle on a sample."""
    B = 48
    b = gen.particles(96, B, 0.05, seed=43, shift_mode=gen.SHIFT_UNIFORM, shift_max=4.0)
    bands = [8, 12, 16, 24, 32, 48]
    h = handle(96, 48, max_batch=B)
    params = mt.Params(bands=bands, n_cand=10, oversample=2, n_alternations=3, shift_window=6)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    sel = [0, 17, 33]
    po = O.align_batch(b.vols[sel], b.ref, dict(L=48, qover=2, L0=8, K=2, ncand=10, bands=bands, iters=1, T=3, W=6))
    for i, p in enumerate(sel):
        assert rot_err_deg(poses[p, :3], po[i, :3]) < TOL_ROT_DEG, (p, rot_err_deg(poses[p, :3], po[i, :3]))
        assert np.abs(poses[p, 3:6] - po[i, 3:6]).max() < 0.1
    errs = [O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) for p in range(B)]
    assert np.median(errs) < 2.0


# ------------------------------------------------------------------ stage 5: upsampled-DFT subpixel
@pytest.mark.parametrize("N,W", [(32, 4), (24, 5), (40, 4), (64, 6)])
def test_translation_upsampled_parity(N, W, prec):
    """matcha_translation_update with upsample = 16 (Guizar-Sicairos refinement, App. C remark iii) vs the oracle's
    separable matrix-multiply DFT in FP64: same integer peak, the same 1/16-grid point (or a neighbour when two grid
    values tie within FP32 rounding: <= 0.1 voxel, north_star's shift tolerance), same c~ at that point."""
    B = 4
    b = gen.particles(N, B, 2.0, seed=45, shift_mode=gen.SHIFT_UNIFORM, shift_max=W - 1.5)
    eul = np.array([O.matrix_to_euler(R) for R in b.truth_R])
    eul[1] += 0.01
    h = handle(N, 8, prec)
    sh, pk = h.translation_update(cuda(b.vols), cuda(b.ref), cuda(eul, h.real), W, upsample=16)
    sh, pk = to_np(sh), to_np(pk)
    eul_used = to_np(cuda(eul, h.real)).astype(np.float64)
    same = 0
    for p in range(B):
        so, po = O.translation_upsampled(b.vols[p], b.ref, eul_used[p], W, 16)
        d = np.abs(sh[p] - so).max()
        assert d <= 0.1, (p, sh[p], so)
        if d < 1e-6:
            same += 1
            assert abs(pk[p] - po) <= (1e-9 if prec == "fp64" else 1e-4) * abs(po), (p, pk[p], po)
        assert np.abs(sh[p] - b.truth_t[p]).max() < 0.3
    assert same >= B - 1


def test_alternation_fractional_shift_upsampled_c1_gpu():
    """SURVEY f3 done-criterion: the c1 fixture with a fractional planted shift reaches <= 0.05 deg and <= 0.01 voxel
    by T = 4 with the upsampled subpixel, and matches the oracle."""
    b = gen.particles(32, 2, float("inf"), seed=12, shift_mode=gen.SHIFT_FIXED, fixed_shift=(1.25, -1.5, 0.75))
    h = handle(32, 8)
    params = mt.Params(bands=[4, 6, 8], n_cand=4, oversample=2, n_alternations=4, shift_window=4, upsample=16)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    po = O.align_batch(b.vols, b.ref, dict(L=8, qover=2, L0=4, K=2, ncand=4, bands=[4, 6, 8], iters=1, T=4, W=4,
                                           ups=16))
    for p in range(2):
        assert rot_err_deg(poses[p, :3], po[p, :3]) < TOL_ROT_DEG
        assert np.abs(poses[p, 3:6] - po[p, 3:6]).max() < 0.1
        assert O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) <= 0.05
        assert np.abs(poses[p, 3:6] - b.truth_t[p]).max() <= 0.01


def test_alternation_c3_shape_upsampled():
    """c3 shape (96^3, SNR 0.05, L0=8 -> 48, T=3, W=6) with the upsampled subpixel: 3 particles of a 32-particle
    batch vs the oracle, and the recovered shifts vs the planted U[-4,4]^3 ones."""
    B = 32
    b = gen.particles(96, B, 0.05, seed=47, shift_mode=gen.SHIFT_UNIFORM, shift_max=4.0)
    bands = [8, 12, 16, 24, 32, 48]
    h = handle(96, 48, max_batch=B)
    params = mt.Params(bands=bands, n_cand=10, oversample=2, n_alternations=3, shift_window=6, upsample=16)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    sel = [0, 13, 31]
    po = O.align_batch(b.vols[sel], b.ref, dict(L=48, qover=2, L0=8, K=2, ncand=10, bands=bands, iters=1, T=3, W=6,
                                                 ups=16))
    for i, p in enumerate(sel):
        assert rot_err_deg(poses[p, :3], po[i, :3]) < TOL_ROT_DEG, (p, rot_err_deg(poses[p, :3], po[i, :3]))
        assert np.abs(poses[p, 3:6] - po[i, 3:6]).max() <= 0.1
    assert np.median(np.abs(poses[:, 3:6] - b.truth_t).max(axis=1)) < 0.5


# ------------------------------------------------------------------ the paper's operating point
def test_paper_operating_point_end_to_end():
    """P:952-953 / P:157: N = 200 boxes, coarse SO(3) grid at L0 = 30 with K = 2 (62 x 124 x 124 = 953k nodes: the
    three-pass global-grid search), N_C = 10, one Newton step per band at {30, 40, 60, L_max} with L_max = 100 (the
    top of the paper's L_max sweep); stage 1 gathers straight from global memory (no 200^3 plane slab fits).
    3 particles at 0 dB (SNR 1.0, the paper's main-text level) vs the FP64 oracle, plus top-K index parity of the
    coarse search under the SURVEY 8(c) separation rule."""
    N, L, bands, nc, B = 200, 100, [30, 40, 60, 100], 10, 3
    b = gen.particles(N, B, 1.0, seed=52)
    h = handle(N, L, max_batch=B)
    params = mt.Params(bands=bands, n_cand=nc, oversample=2)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    po = O.align_batch(b.vols, b.ref, dict(L=L, qover=2, L0=30, K=2, ncand=nc, bands=bands, iters=1, T=1, W=0))
    for p in range(B):
        err = rot_err_deg(poses[p, :3], po[p, :3])
        assert err < TOL_ROT_DEG or abs(poses[p, 6] - po[p, 6]) <= 1e-4 * abs(po[p, 6]), (p, err)
        assert O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) < 0.5
    # the coarse search alone, top-K indices vs the oracle's direct grid
    Fo = O.sh_analysis(b.vols[0], L)
    Ho = O.sh_analysis(b.ref, L)
    Mf = O.corr_full(Fo, Ho, 30)
    Mh = np.stack([O.full_to_half(O.corr_full(Fo, Ho, L), L)])
    eul, sc, idx = h.so3_search(cuda(Mh, h.cplx), L, 30, 2, nc)
    grid = O.grid_eval(Mf, 30, 2)
    all_idx, all_sc, n = O.find_maxima(grid, 100000)
    E0 = O.energy(Fo, Ho, 30)
    idx = to_np(idx)
    compared = 0
    for k in range(nc):
        if topk_index_must_match(all_sc[:n], all_idx[:n], k, grid, E0):
            compared += 1
            assert idx[0, k] == all_idx[k], (k, idx[0, k], all_idx[k])
    assert compared >= 3


# ------------------------------------------------------------------ multi-template + reference update
def _two_template_batch(N, B, snr, seed, cls):
    b = gen.particles(N, B, float("inf"), seed=seed, shift_mode=gen.SHIFT_UNIFORM, shift_max=1.5)
    blobs1 = gen.reference_blobs(seed=0xBEEF)
    ref1 = gen.render(blobs1, N)[0]
    vols = b.vols.copy()
    for p in np.nonzero(cls == 1)[0]:
        vols[p] = gen.render(blobs1, N, R=b.truth_R[p], t=b.truth_t[p])[0]
    if np.isfinite(snr):
        r = np.random.default_rng(seed)
        vols += (r.normal(size=vols.shape) * np.sqrt(b.p_ref / snr)).astype(np.float32)
    return b, vols, np.stack([b.ref, ref1])


@pytest.mark.parametrize("T,W", [(1, 0), (3, 4)])
def test_align_multi_template_parity(T, W, prec):
    """matcha_align_multi (reading C29) vs the oracle: the same template per particle, rotations within
    0.05 deg, shifts within 0.1 voxel; the classes match the planted ones."""
    N, B = 32, 8
    cls = np.array([0, 1, 1, 0, 1, 0, 0, 1])
    b, vols, refs = _two_template_batch(N, B, 1.0, 62, cls)
    h = handle(N, 8, prec, max_batch=5)   # two chunks
    params = mt.Params(bands=[4, 6, 8], n_cand=4, oversample=2, n_alternations=T, shift_window=W)
    poses = to_np(h.align_multi(cuda(vols), cuda(refs), params))
    h.status()
    po = O.align_batch_multi(vols, refs, dict(L=8, qover=2, L0=4, K=2, ncand=4, bands=[4, 6, 8], iters=1, T=T, W=W))
    assert poses[:, 8].astype(int).tolist() == po[:, 8].astype(int).tolist() == cls.tolist()
    for p in range(B):
        assert rot_err_deg(poses[p, :3], po[p, :3]) < TOL_ROT_DEG, p
        assert np.abs(poses[p, 3:6] - po[p, 3:6]).max() < 0.1, p


def test_align_multi_one_template_equals_align_batch():
    b = gen.particles(32, 6, 0.5, seed=63)
    h = handle(32, 8)
    params = mt.Params(bands=[4, 6, 8], n_cand=4)
    p1 = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    pm = to_np(h.align_multi(cuda(b.vols), cuda(b.ref[None]), params))
    assert np.array_equal(p1, pm[:, :8]) and np.all(pm[:, 8] == 0)


def test_reconstruct_parity(prec):
    """matcha_reconstruct (P:1184 half sets; reading C28) vs the oracle's FP64 back-projection, 2 classes,
    shifted poses, an odd first index: elementwise within the FP32 summation bound (FP64: 1e-12)."""
    N, B = 32, 20
    b = gen.particles(N, B, 0.5, seed=64)
    r = np.random.default_rng(64)
    poses = np.zeros((B, 9))
    poses[:, :3] = [O.matrix_to_euler(R) for R in b.truth_R]
    poses[:, 3:6] = r.uniform(-2, 2, (B, 3))
    poses[:, 8] = r.integers(0, 2, B)
    h = handle(N, 8, prec)
    sums, counts = h.reconstruct(cuda(b.vols), cuda(poses, h.real), n_classes=2, class_col=8, first_index=7)
    sums, counts = to_np(sums), to_np(counts)
    poses_used = to_np(cuda(poses, h.real)).astype(np.float64)
    so, co = O.reconstruct(b.vols, poses_used, n_classes=2, class_col=8, first_index=7)
    assert np.array_equal(counts, co)
    bound = np.abs(b.vols).max() * B
    assert np.abs(sums - so).max() <= (1e-12 if prec == "fp64" else 1e-5) * bound, np.abs(sums - so).max() / bound


# ------------------------------------------------------------------ ball-harmonic radial basis
@pytest.mark.parametrize("N,L,lam", [(64, 32, 0.0), (32, 8, 20.0)])
def test_ball_transform_and_corr_parity(N, L, lam, prec):
    """matcha_ball_kmax / matcha_ball_transform / matcha_corr_coeffs_ball (App. A.1; reading C30) vs the
    oracle (independent j_l by the plane-wave integral): identical truncation sets K_l, ball coefficients and the
    rank-|K_l| correlation tensor elementwise."""
    B = 3
    b = gen.particles(N, B, 0.2, seed=72)
    Fo = O.sh_analysis_batch(b.vols, L)
    Ho = O.sh_analysis(b.ref, L)
    h = handle(N, L, prec)
    km, K = h.ball_kmax(lam)
    Ko, _ = O.ball_tables(L, N // 2, lam)
    assert K == Ko.tolist() and km == Ko.max()
    fb = h.ball_transform(cuda(Fo, h.cplx), lam)
    hb = h.ball_transform(cuda(Ho[None], h.cplx), lam)[0]
    M = to_np(h.corr_coeffs_ball(fb, hb, L, lam))
    fb = to_np(fb)
    tol_b = 1e-12 if prec == "fp64" else 2e-6
    Hbo = O.ball_transform(Ho.astype(np.complex64).astype(np.complex128) if prec == "fp32" else Ho, lam)
    for p in range(B):
        Fin = Fo[p].astype(np.complex64).astype(np.complex128) if prec == "fp32" else Fo[p]
        Fbo = O.ball_transform(Fin, lam)
        assert np.abs(fb[p] - Fbo).max() <= tol_b * np.abs(Fbo).max()
        Mo = O.full_to_half(O.corr_ball_full(Fbo, Hbo, N // 2, L, lam), L)
        assert np.abs(M[p] - Mo).max() <= (1e-11 if prec == "fp64" else 1e-5) * np.abs(Mo).max()


def test_align_ball_basis_c2_shape():
    """align_batch with radial = 1 (the paper's ball-harmonic representation with the default cutoff): c2 shape,
    8 particles vs the oracle's ball path, and near the planted rotations."""
    N, L, B = 64, 32, 8
    b = gen.particles(N, B, 0.1, seed=73)
    bands = [8, 12, 16, 24, 32]
    h = handle(N, L, max_batch=B)
    params = mt.Params(bands=bands, n_cand=10, oversample=2, radial=1)
    poses = to_np(h.align_batch(cuda(b.vols), cuda(b.ref), params))
    h.status()
    po = O.align_batch(b.vols, b.ref, dict(L=L, qover=2, L0=8, K=2, ncand=10, bands=bands, iters=1, radial=1))
    for p in range(B):
        assert rot_err_deg(poses[p, :3], po[p, :3]) < TOL_ROT_DEG or abs(poses[p, 6] - po[p, 6]) <= 1e-4 * abs(po[p, 6])
    errs = [O.geodesic_deg_matrix(O.euler_to_matrix(poses[p, :3]), b.truth_R[p]) for p in range(B)]
    assert np.median(errs) < 1.0


def test_align_cuda_graph_replay_bitwise():
    """matcha_set_graphs: repeated identical align_batch calls are captured once and replayed as a CUDA graph; the
    poses are bitwise those of the eager path (chunked, translating)."""
    b = gen.particles(32, 20, 0.5, seed=81, shift_mode=gen.SHIFT_UNIFORM, shift_max=2.0)
    vols, ref = cuda(b.vols), cuda(b.ref)
    params = mt.Params(bands=[4, 6, 8], n_cand=4, n_alternations=2, shift_window=4)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        h = handle(32, 8, max_batch=8)
        eager = to_np(h.align_batch(vols, ref, params))
        h.set_graphs(True)
        out = torch.empty((20, 8), device=DEV)
        n0 = h.launches
        for _ in range(3):  # eager (key recorded), capture + replay, replay
            h.align_batch(vols, ref, params, out=out)
            s.synchronize()
            assert np.array_equal(to_np(out), eager)
        assert h.launches - n0 > 0
        h.set_graphs(False)


def test_synth_particles_matches_host_generator():
    """matcha_synth_particles reproduces gen/gen.c's seeded workload on the device (same Philox counters and phantom):
    poses equal to rounding, volumes to the last float ulp (device vs host exp/log), noisy and shifted."""
    N, B = 32, 5
    h = handle(N, 8)
    for snr, smax in ((0.1, 0.0), (float("inf"), 3.0)):
        vols, truth = h.synth_particles(B, snr, seed=17, first_index=40, shift_max=smax)
        kw = dict(shift_mode=gen.SHIFT_UNIFORM, shift_max=smax) if smax > 0 else {}
        hb = gen.particles(N, B, snr, seed=17, first=40, **kw)
        truth = to_np(truth)
        assert np.abs(truth[:, :9].reshape(B, 3, 3) - hb.truth_R).max() < 1e-14
        assert np.abs(truth[:, 9:] - hb.truth_t).max() < 1e-14
        v = to_np(vols)
        assert np.abs(v - hb.vols).max() <= 2e-6 * np.abs(hb.vols).max()
