#!/usr/bin/env python
"""bench.py -- particles aligned/s (box 64^3, L0=8 -> L=32, device-timed) on 1..8 B200.

A "step" is one pass of the whole hot path over one batch of synthetic particles: reference
coefficients (rank 0, broadcast over NCCL when N>1), then per particle stage 1 (shell SH analysis),
stage 2 (Wigner coefficient tensor), stage 3 (coarse SO(3) search), stage 4 (frequency-marching
Newton, final C_{L_J}, argmax), pose gather (all_gather over NCCL when N>1).  Weak scaling: every
rank aligns its own --particles (default 1,000 = BASELINE configs[1], "c2").

    python bench.py [--gpus N --steps K --warmup W] [--impl matcha|reference] [--config c2|c3|c4|c5]
    torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line.  See DESIGN.md "Measurement" for the roofline arithmetic.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particles aligned/s (box 64³, L0=8→L=32, device-timed)"
CONFIGS = {
    # BASELINE.json configs[1] (c2) -- the metric's workload; c4 = the same shape at STA scale
    "c2": dict(N=64, L=32, bands=[8, 12, 16, 24, 32], ncand=10, K=2, snr=0.1, particles=1000, iters=1),
    "c4": dict(N=64, L=32, bands=[8, 12, 16, 24, 32], ncand=10, K=2, snr=0.1, particles=12500, iters=1),
    # configs[4] (c5), high-bandwidth Newton stress
    "c5": dict(N=128, L=64, bands=[12, 16, 24, 32, 48, 64], ncand=16, K=2, snr=0.1, particles=1000, iters=1),
    # configs[2] (c3): 96^3, SNR 0.05, shifts U[-4,4]^3, T = 3 alternations with the FFT translation update
    # (W = 6); 1,000 particles per rank (the 10,000-particle job is 10 such steps)
    "c3": dict(N=96, L=48, bands=[8, 12, 16, 24, 32, 48], ncand=10, K=2, snr=0.05, particles=1000, iters=1,
               T=3, W=6, shift_max=4.0),
    # c3 with the upsampled-DFT subpixel refinement (kappa = 16 over +-1.5 voxel, App. C remark iii)
    "c3u": dict(N=96, L=48, bands=[8, 12, 16, 24, 32, 48], ncand=10, K=2, snr=0.05, particles=1000, iters=1,
                T=3, W=6, shift_max=4.0, ups=16),
    # the paper's operating point: N = 200, coarse grid at L0 = 30 with K = 2
    # (953k nodes), N_C = 10, one Newton step per band at {30, 40, 60, L_max}, L_max = 100; 0 dB (SNR 1.0)
    "paper": dict(N=200, L=100, bands=[30, 40, 60, 100], ncand=10, K=2, snr=1.0, particles=500, iters=1),
    # c2 with the paper's ball-harmonic radial basis (eigenvalue cutoff pi (R - 1/2))
    "c2b": dict(N=64, L=32, bands=[8, 12, 16, 24, 32], ncand=10, K=2, snr=0.1, particles=1000, iters=1, radial=1),
    # one multi-template STA iteration at c2 shape: alignment against 2 templates + the half-map update
    "c2m": dict(N=64, L=32, bands=[8, 12, 16, 24, 32], ncand=10, K=2, snr=0.1, particles=1000, iters=1, templates=2),
    # configs[0] (c1) rotation part, small
    "c1": dict(N=32, L=8, bands=[4, 6, 8], ncand=4, K=2, snr=float("inf"), particles=64, iters=1),
}
SEED = 1


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def mh(L):
    return (L + 1) * (L + 2) * (4 * L + 3) // 6


def ncoef(L):
    return (L + 1) * (L + 2) // 2


def stage_work(c):
    """Algorithmic (flops, bytes) per particle for each kernel."""
    N, L, K, nc = c["N"], c["L"], c["K"], c["ncand"]
    R, Lq = N // 2, 2 * L
    nth, nph = Lq + 1, 2 * Lq + 2
    Jh, Kh = (nth + 1) // 2, (nph // 2 - 1) // 2
    samples = R * nth * nph
    # SURVEY 8(d)'s accounting (15.1 MFLOP per particle at c2): a1 trilinear ~21 flop/sample; a2 the real-data
    # folded ring DFT ~(L+1)/2 flop/sample and the Legendre contraction 8 flop per (shell, node pair, (l, m))
    sh_fl = 21 * samples + samples * (L + 1) // 2 + R * Jh * ncoef(L) * 8
    sh_by = 4 * N ** 3 + 8 * ncoef(L) * R
    corr_fl = 8 * R * mh(L)
    corr_by = 8 * ncoef(L) * R + 8 * mh(L)
    L0 = c["bands"][0]
    nb, na = K * (L0 + 1), 2 * K * (L0 + 1)
    srch_fl = nb * (mh(L0) * 12 + (L0 + 1) * na * (2 * L0 + 1) * 8 + na * na * L0 * 4 + na * na * 26)
    srch_by = 8 * mh(L0)
    nw_fl = sum(c["iters"] * mh(Lj) * nc * 28 for Lj in c["bands"]) + mh(c["bands"][-1]) * nc * 8
    nw_by = sum(c["iters"] * 8 * mh(Lj) for Lj in c["bands"]) + 8 * mh(c["bands"][-1])
    T = c.get("T", 1)
    nt = c.get("templates", 1)
    if nt > 1:
        corr_fl, corr_by = nt * corr_fl, nt * corr_by  # M per template
    work = {"sh_analysis": (T * sh_fl, T * sh_by), "corr_coeffs": (T * corr_fl, T * corr_by),
            "so3_search": (T * srch_fl, T * srch_by), "newton_refine": (T * nw_fl, T * nw_by),
            "gather_poses": (0, 48),
            # f4 half-map update: ~30 flop per (voxel, particle) (rotation + trilinear), the particle read once
            "reconstruct": (30 * N ** 3, 4 * N ** 3),
            # f2 radial transform: 8 flop per (shell, (l, m), k); F read, f^ written
            "ball_transform": (8 * R * ncoef(L) * R, 16 * ncoef(L) * R)}
    if nt > 1:
        for k in ("so3_search", "newton_refine"):
            work[k] = (nt * work[k][0], nt * work[k][1])
    if c.get("W", 0) > 0:
        # a11-a13 per alternation (k_trans.cu, no FFT library): rho~ = 2-D R2C of every z-plane of the rotated
        # reference (rotation fused: ~30 flop/voxel, 2.5 N^2 log2 N^2 flop per plane), the z correlation of the plane
        # spectra onto the w' = 2W+3 window (8 flop per complex MAC, N^2 H w' MACs), the (x, y) window inverse;
        # once per particle f~ (the particle's plane spectra).  Bytes: f~ read + rho~ written and read + Y1 written
        # and read per alternation; f read and f~ written once.
        n3, H, wp = N ** 3, N // 2 + 1, 2 * c["W"] + 3
        lg2 = 2 * np.log2(N)
        plane_fft = 2.5 * n3 * lg2
        alt_fl = 30 * n3 + plane_fft + 8 * N * N * H * wp + 8 * wp * (N * H * wp + N * wp * wp)
        alt_by = 3 * 8 * N * N * H + 2 * 16 * wp * N * H
        once_fl, once_by = plane_fft, 4 * n3 + 8 * N * N * H
        if c.get("ups"):
            # f3: z FFTs of f~ and rho~ -> X, then the three matrix-multiply DFTs onto the U^3 grid
            U = 2 * int(np.ceil(1.5 * c["ups"])) + 1
            alt_fl += 2 * 5 * N * N * H * np.log2(N) + 6 * N * N * H + 8 * N * (N * H * U + N * U * U) + 4 * N * U ** 3
            alt_by += 4 * 8 * N * N * H + 2 * 8 * N * U * U
        work["translation_update"] = (int(T * alt_fl + once_fl), int(T * alt_by + once_by))
    return work


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.rows = []
        self.t0 = self.t1 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(index)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def mark(self, start):
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        rows = [r for t, r in self.rows if self.t0 is not None and self.t0 - 0.2 <= t <= (self.t1 or t) + 0.2]
        if not rows:
            rows = [r for _, r in self.rows]
        rows = [r for r in rows if len(r) >= 8]
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def make_batch(c, rank, world, P):
    import gen
    if c.get("shift_max"):
        return gen.particles(c["N"], P, c["snr"], seed=SEED, first=rank * P, shift_mode=gen.SHIFT_UNIFORM,
                             shift_max=c["shift_max"])
    return gen.particles(c["N"], P, c["snr"], seed=SEED, first=rank * P)


def oracle_params(c):
    return dict(L=c["L"], qover=2, L0=c["bands"][0], K=c["K"], ncand=c["ncand"], bands=c["bands"],
                iters=c["iters"], T=c.get("T", 1), W=c.get("W", 0), ups=c.get("ups", 0), radial=c.get("radial", 0))


def template_refs(c, ref):
    """f4 workloads: the reference plus further phantoms of the same recipe (Philox keys 0xBEEF + k)."""
    import gen as G
    return np.stack([ref] + [G.render(G.reference_blobs(seed=0xBEEF + k), c["N"])[0]
                             for k in range(c.get("templates", 1) - 1)])


def time_oracle(vols, ref, c, n, nthreads):
    import oracle as O
    t = time.perf_counter()
    if c.get("templates", 1) > 1:
        poses = O.align_batch_multi(vols[:n], template_refs(c, ref), oracle_params(c), nthreads=nthreads)
        O.reconstruct(vols[:n], poses, n_classes=c["templates"], class_col=8)
    else:
        O.align_batch(vols[:n], ref, oracle_params(c), nthreads=nthreads)
    return time.perf_counter() - t


def cpu_baseline(batch, c, budget_s=20.0):
    """The FP64 oracle as it stands, on this host's cores, on a bounded sample of the same workload."""
    cores = os.cpu_count() or 1
    # calibrate on one particle per thread (the pool's real throughput, not 1-thread time x cores)
    n0 = min(cores, len(batch.vols))
    t0 = time_oracle(batch.vols, batch.ref, c, n0, cores)
    n = int(max(n0, min(len(batch.vols), budget_s * n0 / max(t0, 1e-3))))
    n = max(n0, (n // n0) * n0)
    t = t0 if n == n0 else time_oracle(batch.vols, batch.ref, c, n, cores)
    return {"value": n / t, "unit": "particles/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} of the {len(batch.vols)} {c['N']}^3 particles of this workload (same seed), "
                      f"std::thread pool of {cores}, FP64 C++ oracle (oracle/oracle.cpp)"}


def run_reference(args, c, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host cores, rank 0 only."""
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    batch = make_batch(c, 0, 1, min(c["particles"], 4096))
    n0 = min(cores, len(batch.vols))
    t0 = time_oracle(batch.vols, batch.ref, c, n0, cores)  # one particle per pool thread: calibration
    per_step_budget = 150.0 / max(1, args.steps + args.warmup)
    S = int(max(n0, min(len(batch.vols), per_step_budget * n0 / max(t0, 1e-3))))
    for _ in range(args.warmup):
        time_oracle(batch.vols, batch.ref, c, S, cores)
    t = 0.0
    for _ in range(args.steps):
        t += time_oracle(batch.vols, batch.ref, c, S, cores)
    value = S * args.steps / t
    sample = (f"{S} particles per step of the {c['N']}^3 workload (same seed), std::thread pool of {cores}, "
              "FP64 C++ oracle")
    out = {"metric": metric_of(args.config, c), "value": value, "unit": "particles/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": workload_of(args.config, c, c["particles"]),
                      "particles_per_rank": c["particles"], "parallelism": "dp1",
                      "oracle_particles_per_step": S},
           "cpu_baseline": {"value": value, "unit": "particles/s", "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def workload_of(name, c, P):
    """The workload string both arms print (the matcha arm's config.workload; the reference arm times the oracle on
    a bounded sample of the same workload)."""
    return (f"{name}: {P} particles/rank of {c['N']}^3, SNR {c['snr']}, "
            f"L0={c['bands'][0]}->L={c['L']} bands {c['bands']}, N_C={c['ncand']}, "
            f"K={c['K']}, 1 Newton step/band, "
            + (f"T={c['T']} alternations with the FFT translation update (W={c['W']}, "
               + (f"upsampled-DFT subpixel kappa={c['ups']}" if c.get("ups") else "parabolic subpixel")
               + f"), shifts U[-{c['shift_max']:g},{c['shift_max']:g}]^3" if c.get("T", 1) > 1 else "rotation only")
            + (", ball-harmonic radial basis (radial=1)" if c.get("radial") else "")
            + (f", {c['templates']} templates + half-map reference update per step"
               if c.get("templates", 1) > 1 else ""))


def metric_of(name, c):
    """BASELINE's metric for its workload (c2/c4); the same measure named for the other configs."""
    if name in ("c2", "c4"):
        return METRIC
    alt = f", T={c['T']} alternations" if c.get("T", 1) > 1 else ""
    if c.get("radial"):
        alt += ", ball-harmonic radial basis"
    if c.get("templates", 1) > 1:
        return (f"particles refined/s (box {c['N']}³, L0={c['bands'][0]}→L={c['L']}, {c['templates']} templates + "
                "half-map update, device-timed)")
    if c.get("ups"):
        alt += f", upsampled subpixel kappa={c['ups']}"
    return f"particles aligned/s (box {c['N']}³, L0={c['bands'][0]}→L={c['L']}{alt}, device-timed)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="matcha", choices=["matcha", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--particles", type=int, default=None, help="particles per rank (weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference" or os.environ.get("BENCH_ALLOW_SHORT"), "W >= 3"
    c = dict(CONFIGS[args.config])
    if args.particles:
        c["particles"] = args.particles

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, c, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2603_15285_b200 as mt

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    P = c["particles"]
    batch = make_batch(c, rank, world, P)
    vols_host = torch.from_numpy(batch.vols).pin_memory()
    ref_host = torch.from_numpy(batch.ref).pin_memory()
    vols = vols_host.to(dev)
    ref = ref_host.to(dev)
    h = mt.Handle(N=c["N"], L_max=c["L"], quad_oversample=2, max_batch=P)
    params = mt.Params(bands=c["bands"], n_cand=c["ncand"], oversample=c["K"], newton_iters=c["iters"],
                       n_alternations=c.get("T", 1), shift_window=c.get("W", 0), upsample=c.get("ups", 0),
                       radial=c.get("radial", 0))
    from paper_2603_15285_b200 import dist as D
    H = torch.empty((ncoef(c["L"]), c["N"] // 2), dtype=torch.complex64, device=dev)
    counts = [P] * world

    nt = c.get("templates", 1)
    if nt > 1:
        # f4: the templates are the reference and further phantoms of the same recipe (other Philox keys)
        refs = torch.from_numpy(template_refs(c, batch.ref)).to(dev)
        Hs = torch.empty((nt, ncoef(c["L"]), c["N"] // 2), dtype=torch.complex64, device=dev)

    def step():
        if nt > 1:
            # f4: multi-template alignment + the half-map reference update (NCCL all-reduce of 2 T N^3 sums)
            D.sta_step(h, vols, refs, params, Hs, rank, first_index=rank * P, counts=counts)
            return
        # rank 0: reference coefficients (stage a3) -> NCCL broadcast (140 KiB at c2) -> every rank aligns its
        # shard -> NCCL all_gather of the poses (32 B per particle)
        D.align_step(h, vols, ref, params, H, rank, counts=counts)

    for _ in range(args.warmup):
        step()
    h.status()
    torch.cuda.synchronize()

    clk = ClockSampler(local)
    time.sleep(0.3)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = h.launches
    h.profile_begin()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark(True)
    e0.record(s)
    for _ in range(args.steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    clk.mark(False)
    if world > 1:
        dist.barrier()
    stages = h.profile_end()
    n_launch = h.launches - n_launch0
    ms = D.max_over_ranks(e0.elapsed_time(e1), device=dev)
    clocks = clk.stop()
    h.status()

    value = P * world * args.steps / (ms / 1e3)

    # ---- end to end through the public API on host buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e and nt == 1:
        # the public host-buffer call in chunks of P/4 particles: the H2D copy of chunk c+1 (second stream) overlaps
        # the compute of chunk c (matcha_align_batch_host's double buffering)
        h = mt.Handle(N=c["N"], L_max=c["L"], quad_oversample=2, max_batch=max(1, (P + 3) // 4))
        out_host = torch.empty((P, 8), dtype=torch.float32).pin_memory()
        for _ in range(2):
            h.align_batch_host(vols_host, ref_host, params, out=out_host)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ksteps = max(3, min(args.steps, 10))
        for _ in range(ksteps):
            h.align_batch_host(vols_host, ref_host, params, out=out_host)
        dt = D.max_over_ranks(time.perf_counter() - t0, device=dev)
        e2e = {"value": P * world * ksteps / dt, "unit": "particles/s",
               "h2d_bytes_per_step": int(vols_host.numel() * 4 + ref_host.numel() * 4),
               "d2h_bytes_per_step": int(out_host.numel() * 4)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (live CUDA-event timing of each stage launch)
    pk, src = peaks()
    sm_max = (clocks or {}).get("sm_max_mhz") or pk.get("sm_max_mhz", 1965.0)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = nsm * 128 * 2 * sm_max * 1e6 / 1e12  # FP32 FFMA pipe, TFLOP/s
    hbm_peak = pk["hbm_gbs"]
    work = stage_work(c)
    tot_ms = sum(v[0] for v in stages.values())
    dom = max(stages, key=lambda k: stages[k][0])
    dms, dn = stages[dom]
    # units the dominant stage processed in the timed region (sh_analysis also analyses the reference)
    units = args.steps * (P + (1 if dom == "sh_analysis" else 0))
    fl, by = work[dom]
    t_stage = dms / 1e3
    t_alu, t_hbm = fl / (alu_peak * 1e12), by / (hbm_peak * 1e9)
    traffic = traffic_pp = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        tr = json.load(open(tp)).get(args.config, {}).get(dom)
        if isinstance(tr, dict) and tr.get("bytes_per_particle") is not None:
            traffic_pp = tr["bytes_per_particle"]
            traffic = traffic_pp * units / dn  # DRAM bytes per launch, like achieved
    if t_alu >= t_hbm:
        achieved = fl * units / t_stage / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": achieved / alu_peak, "traffic": traffic}
    else:
        achieved = by * units / t_stage / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": traffic}
    # every stage against its own bound on the same model (the north_star evaluation kernel is newton_refine)
    per_stage = {}
    for k, (ms_k, n_k) in stages.items():
        if k not in work or ms_k <= 0:
            continue
        u_k = args.steps * (P + (1 if k == "sh_analysis" else 0))
        fl_k, by_k = work[k]
        if fl_k / (alu_peak * 1e12) >= by_k / (hbm_peak * 1e9):
            per_stage[k] = {"bound": "alu", "frac": fl_k * u_k / (ms_k / 1e3) / 1e12 / alu_peak}
        else:
            per_stage[k] = {"bound": "hbm", "frac": by_k * u_k / (ms_k / 1e3) / 1e9 / hbm_peak}
    roof["stages"] = per_stage
    roof.update({"kernel": dom, "share_of_step": dms / tot_ms if tot_ms else None,
                 "peak_source": (f"{nsm} SMs x 128 FP32 lanes x 2 x {sm_max:.0f} MHz (guide unit counts)"
                                 if roof["bound"] == "alu" else f"MEASURED_PEAKS.json hbm_gbs ({src})"),
                 "launches": dn, "avg_launch_ms": dms / dn,
                 "work_per_particle": {"flop": fl, "bytes": by},
                 "traffic_unit": "DRAM bytes per launch of the stage (ncu dram__bytes_read+write of its kernels "
                                 "per particle, profiles/traffic.json, x particles per launch)",
                 "traffic_per_particle": traffic_pp,
                 "algorithmic_bytes_per_launch": by * units / dn,
                 "hbm_gbs_achieved": by * units / t_stage / 1e9,
                 "alu_tflops_achieved": fl * units / t_stage / 1e12,
                 "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()}})

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(batch, c)

    out = {"metric": metric_of(args.config, c), "value": value, "unit": "particles/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": {"workload": workload_of(args.config, c, P),
                      "particles_per_rank": P, "parallelism": f"dp{world}",
                      "l2": f"inputs larger than L2 ({P * c['N'] ** 3 * 4 / 2**30:.2f} GiB per rank resident)"},
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": n_launch, "clocks": clocks}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
