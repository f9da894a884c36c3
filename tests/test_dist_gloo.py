"""Multi-process (world_size 2, gloo, CPU) tests of the data-parallel host logic of bench.py / dist.py:
sharding covers every particle exactly once, the reference coefficients are broadcast from rank 0, poses are
gathered in global particle order (ragged shards too), and the elapsed time is the max over ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_15285_b200 import dist as D


def test_shard_covers_all_particles_once():
    for P in (0, 1, 7, 1000, 100001):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = D.shard(P, world, r)
                assert 0 <= a <= b <= P
                seen.extend(range(a, b))
            assert seen == list(range(P))
            sizes = [D.shard(P, world, r)[1] - D.shard(P, world, r)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


class FakeHandle:
    """CPU test double with the Handle call signatures: encodes inputs into the outputs."""

    def sh_analysis(self, vols, out):
        out.copy_(torch.full_like(out, complex(float(vols.sum()), 1.0)))
        return out

    def align_batch(self, vols, ref, params, ref_coeffs=None):
        # the library's contract: a translation update (shift_window > 0) needs the reference volume
        if params is not None and params.shift_window > 0 and ref is None:
            raise RuntimeError("matcha WINDOW: shift window needs ref")
        n = vols.shape[0]
        poses = torch.zeros((n, 8), dtype=torch.float32)
        poses[:, 0] = vols.reshape(n, -1)[:, 0]          # global particle id planted in voxel 0
        poses[:, 6] = float(torch.view_as_real(ref_coeffs).sum())
        poses[:, 7] = -1.0 if ref is None else float(ref.sum())  # the volume the translation update would rotate
        return poses


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _Params:
    def __init__(self, T, W):
        self.n_alternations = T
        self.shift_window = W


def _worker(rank, world, port, P, q, T=1, W=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = D.shard(P, world, rank)
        vols = torch.zeros((b - a, 4, 4, 4))
        vols.reshape(b - a, -1)[:, 0] = torch.arange(a, b, dtype=torch.float32)
        # rank 1 starts with another reference volume: with translation (W > 0) it must receive rank 0's
        ref = torch.full((4, 4, 4), 0.5 if rank == 0 else 9.0)
        H = torch.zeros((3, 2), dtype=torch.complex64)  # rank 1 starts with zeros: must receive rank 0's
        poses = D.align_step(FakeHandle(), vols, ref, _Params(T, W) if T else None, H, rank)
        t = D.max_over_ranks(float(rank + 1))
        # plain Python values only: a tensor would travel as a shared-memory handle that dies with this process
        q.put((rank, poses[:, 0].tolist(), poses[:, 6].tolist(), torch.view_as_real(H).tolist(), t,
               poses[:, 7].tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P,T,W", [(10, 0, 0), (7, 1, 0), (7, 3, 2), (7, 1, 2), (7, 3, 0)])
def test_align_step_world2_gloo(P, T, W):
    """The translation predicate is the library's (shift_window > 0), not n_alternations > 1: T=1 with W>0 still
    translates (the reference volume is broadcast), T>1 with W=0 is rotation only."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, P, q, T, W)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    expect_H = torch.full((3, 2), complex(0.5 * 64, 1.0), dtype=torch.complex64)
    for rank, ids, checks, H, t, refsum in res:
        assert ids == [float(i) for i in range(P)]                  # gathered in global order
        assert torch.equal(torch.view_as_complex(torch.tensor(H)), expect_H)  # broadcast from rank 0
        assert all(abs(c - float(torch.view_as_real(expect_H).sum())) < 1e-3 for c in checks)
        assert t == 2.0                                             # max over ranks
        # rotation only: no reference volume is passed; translating: rank 0's volume on every rank
        assert refsum == [-1.0 if (not T or W == 0) else 0.5 * 64] * P


class FakeReconHandle:
    """CPU double of Handle.reconstruct: sums = (global index) planted per particle, counts per half."""

    def reconstruct(self, vols, poses, n_classes=1, class_col=-1, first_index=0):
        n = vols.shape[0]
        sums = torch.zeros((n_classes, 2, 2, 2, 2), dtype=torch.float64)
        counts = torch.zeros((n_classes, 2), dtype=torch.int32)
        for p in range(n):
            g = first_index + p
            sums[0, g % 2] += float(g)
            counts[0, g % 2] += 1
        return sums, counts


def _recon_worker(rank, world, port, P, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = D.shard(P, world, rank)
        avg, counts = D.reconstruct_step(FakeReconHandle(), torch.zeros((b - a, 2, 2, 2)), torch.zeros((b - a, 8)),
                                         first_index=a)
        q.put((rank, avg[0, :, 0, 0, 0].tolist(), counts.tolist()))
    finally:
        dist.destroy_process_group()


def test_reconstruct_step_world2_gloo():
    """half-map sums and counts are all-reduced across ranks before the division (global half sets)."""
    P = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_recon_worker, args=(r, 2, port, P, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    even = [g for g in range(P) if g % 2 == 0]
    odd = [g for g in range(P) if g % 2 == 1]
    for rank, avg, counts in res:
        assert counts == [[len(even), len(odd)]]
        assert abs(avg[0] - np.mean(even)) < 1e-12 and abs(avg[1] - np.mean(odd)) < 1e-12
