"""Data-parallel driver over particles: one process per GPU, torch.distributed for plumbing.

The path shards naturally -- particles are independent -- so there is no exchange inside it.  The collectives
(NCCL over NVLink on B200; any backend works, the CPU tests use gloo):
  1. broadcast of the reference coefficients H (complex [ncoef][R], 140 KiB at 64^3/L=32) from rank 0;
  2. all_gather of the poses (8 reals = 32 B per particle in FP32);
  3. (the reference update after an alignment pass) all_reduce of the half-map sums (2 N^3 reals per
     class) and counts -- the only N^3 exchange of the domain.
Rank r of G owns the contiguous particle range [floor(r P/G), floor((r+1) P/G)).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def shard(P: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous particle range of `rank` (SURVEY 8(e) partitioning)."""
    return (P * rank) // world, (P * (rank + 1)) // world


def broadcast_ref_coeffs(H: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Reference coefficients computed on `src` are broadcast in place (complex tensors are sent as real views)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(torch.view_as_real(H) if H.is_complex() else H, src=src, group=group)
    return H


def gather_poses(poses: torch.Tensor, counts: Optional[list[int]] = None, group=None) -> torch.Tensor:
    """All-gather per-rank pose blocks [n_r, 8] into [sum n_r, 8] in rank order (ragged shards padded)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return poses
    world = dist.get_world_size(group)
    if counts is None:
        n = torch.tensor([poses.shape[0]], device=poses.device, dtype=torch.int64)
        alln = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(alln, n, group=group)
        counts = [int(x.item()) for x in alln]
    mx = max(counts)
    buf = torch.zeros((mx, poses.shape[1]), dtype=poses.dtype, device=poses.device)
    buf[: poses.shape[0]] = poses
    out = torch.empty((mx * world, poses.shape[1]), dtype=poses.dtype, device=poses.device)
    if poses.is_cuda:
        dist.all_gather_into_tensor(out, buf, group=group)
    else:
        parts = list(out.chunk(world))
        dist.all_gather(parts, buf, group=group)
    return torch.cat([out[r * mx: r * mx + counts[r]] for r in range(world)])


def max_over_ranks(x: float, device=None, group=None) -> float:
    """Elapsed time of a multi-GPU run = max over ranks (device-timed by each rank)."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def align_step(handle, vols_local: torch.Tensor, ref: torch.Tensor, params, H: torch.Tensor,
               rank: int, group=None, counts: Optional[list[int]] = None) -> torch.Tensor:
    """One data-parallel step: rank 0 analyses the reference, H is broadcast, every rank aligns its shard with
    the shared H, the poses are gathered.  `handle` is a paper_2603_15285_b200.Handle (or a test double)."""
    if rank == 0:
        handle.sh_analysis(ref[None], out=H[None])
    broadcast_ref_coeffs(H, src=0, group=group)
    # the library translates iff shift_window > 0 (include/matcha.h, matcha_params_t.shift_window)
    translate = getattr(params, "shift_window", 0) > 0
    if translate:
        # the translation update (App. C) rotates the reference volume itself: rank 0's copy goes to every rank
        broadcast_ref_coeffs(ref, src=0, group=group)
    poses = handle.align_batch(vols_local, ref if translate else None, params, ref_coeffs=H)
    return gather_poses(poses, counts=counts, group=group)


def reconstruct_step(handle, vols_local: torch.Tensor, poses_local: torch.Tensor, first_index: int,
                     n_classes: int = 1, class_col: int = -1, group=None):
    """Reference update of subtomogram averaging (P:1184 half-set split): every rank sums its shard's aligned
    particles per (class, half set) with the library kernel, the sums and counts are all-reduced, and the half maps
    are the ratio (classes/halves without particles stay 0).  -> (half maps [n_classes, 2, N, N, N], counts)."""
    sums, counts = handle.reconstruct(vols_local, poses_local, n_classes=n_classes, class_col=class_col,
                                      first_index=first_index)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(sums, group=group)
        dist.all_reduce(counts, group=group)
    c = counts.to(sums.dtype).clamp(min=1).reshape(n_classes, 2, 1, 1, 1)
    return sums / c, counts


def sta_step(handle, vols_local: torch.Tensor, refs: torch.Tensor, params, Hs: torch.Tensor, rank: int,
             first_index: int, group=None, counts=None):
    """One iteration of multi-template subtomogram averaging: rank 0 analyses the T
    templates, the coefficients (and, when translating, the template volumes) are broadcast, every rank aligns its
    shard against all templates (matcha_align_multi), the half maps of every class are summed per rank and
    all-reduced (reconstruct_step), the poses gathered.  -> (poses [P, 9], half maps [T, 2, N, N, N], counts)."""
    nt = refs.shape[0]
    if rank == 0:
        handle.sh_analysis(refs, out=Hs)
    broadcast_ref_coeffs(Hs, src=0, group=group)
    translate = getattr(params, "shift_window", 0) > 0
    if translate:
        broadcast_ref_coeffs(refs, src=0, group=group)
    poses = handle.align_multi(vols_local, refs if translate else None, params, ref_coeffs=Hs)
    maps, cnt = reconstruct_step(handle, vols_local, poses, first_index, n_classes=nt, class_col=8, group=group)
    return gather_poses(poses, counts=counts, group=group), maps, cnt
