"""Summarise a round's GPU evidence into profiles/<tag>_summary.md (+ traffic.json for bench.py).

usage: python scripts/summarize_profile.py <tag>   (reads gpurun_out/<tag>_{bench.json,launches.csv,full.ncu-rep})
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

tag = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)
out = []

bj = os.path.join(G, f"{tag}_bench.json")
bench = None
if os.path.exists(bj):
    lines = [l for l in open(bj).read().splitlines() if l.strip().startswith("{")]
    if lines:
        bench = json.loads(lines[-1])
        shutil.copy(bj, os.path.join(P, f"{tag}_bench.json"))
        out.append(f"## bench.py (default: c2, 1 GPU)\n\n- value **{bench['value']:.0f} {bench['unit']}**, "
                   f"{bench['ms_per_step']:.3f} ms/step, e2e {bench['e2e']['value']:.0f} (host buffers, PCIe H2D "
                   f"{bench['e2e']['h2d_bytes_per_step'] / 1e9:.2f} GB/step)")
        r = bench["roofline"]
        out.append(f"- dominant kernel `{r['kernel']}` ({100 * r['share_of_step']:.1f} % of the step): "
                   f"{r['achieved']:.2f} {r['unit']} of {r['peak']:.1f} ({r['bound']}) = {100 * r['frac']:.1f} %; "
                   f"{r['hbm_gbs_achieved']:.0f} GB/s algorithmic")
        out.append("- per-stage device ms/step (CUDA events on the launching stream): " + ", ".join(
            f"{k} {v:.3f}" for k, v in r["stages_ms_per_step"].items()))
        if bench.get("cpu_baseline"):
            cb = bench["cpu_baseline"]
            out.append(f"- cpu_baseline (FP64 oracle): {cb['value']:.1f} particles/s on {cb['cores']} cores")
        out.append(f"- clocks: {bench.get('clocks')}\n")

lc = os.path.join(G, f"{tag}_launches.csv")
if os.path.exists(lc):
    shutil.copy(lc, os.path.join(P, f"{tag}_launches.csv"))
    rows = list(csv.reader(open(lc)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[hdr["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        u = r[hdr["Metric Unit"]]
        us = v / 1e3 if u == "nsecond" else v * 1e3 if u == "msecond" else v / 1e6 if u == "psecond" else v
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values()) or 1
    out.append("## ncu launch list (gpu__time_duration, cold-cache, serialised): share of GPU time\n")
    out.append("| kernel | launches | total µs | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f} % |")
    out.append("")

import glob
reps = sorted(glob.glob(os.path.join(G, f"{tag}_full*.ncu-rep")))
traffic = {}
header_done = False
for rep in reps:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
    if not header_done:
        header_done = True
        out.append("## ncu --set full (one launch per kernel)\n")
        out.append("| kernel | " + " | ".join(w.replace(".avg.pct_of_peak_sustained_active", " %").replace(".sum", "")
                                             for w in want) + " |")
        out.append("|" + "---|" * (len(want) + 1))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        vals = []
        for w in want:
            vals.append(r[hdr.index(w)] if w in hdr else "n/a")
        out.append(f"| `{name}` | " + " | ".join(vals) + " |")
        try:
            sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[hdr.index("dram__bytes_read.sum")]) * sc.get(rows[1][hdr.index("dram__bytes_read.sum")], 1)
            wr = float(r[hdr.index("dram__bytes_write.sum")]) * sc.get(rows[1][hdr.index("dram__bytes_write.sum")], 1)
            scale = 1.0
            key = "sh_analysis" if "k_sh" in name else "newton_refine" if "newton" in name else \
                "so3_search" if ("search" in name or "so3" in name) else "corr_coeffs" if "corr" in name else name
            # particles in the captured launch: every captured launch (round 2: stage 1 too, one ring sub-batch per
            # c2 chunk) covers the whole 1,000-particle batch
            per = int(os.environ.get("PARTICLES_PER_LAUNCH", "1000"))
            traffic.setdefault(key, 0.0)
            traffic[key] += (rd + wr) * scale / per
        except (ValueError, IndexError):
            pass
    shutil.copy(rep, os.path.join(P, os.path.basename(rep)))
if header_done:
    out.append("\n(dram units as printed by ncu; every captured launch covers the 1,000-particle batch)\n")
    out.append("DRAM traffic per particle (bytes, from the captures above): " +
               ", ".join(f"{k} {v:.0f}" for k, v in traffic.items()) + "\n")
    json.dump({"c2": {k: {"bytes_per_particle": v, "source": f"profiles/{tag}_full_*.ncu-rep dram__bytes_read+write"}
                      for k, v in traffic.items()}}, open(os.path.join(P, "traffic.json"), "w"), indent=1)

# warm-cache DRAM traffic (--cache-control none): preferred for traffic.json when present
warm = {}
for f in sorted(glob.glob(os.path.join(G, f"{tag}_warm_*.csv"))):
    kname = os.path.basename(f)[len(tag) + 6:-4]
    vals = {}
    for r in csv.reader(open(f)):
        if len(r) > 12 and r[-3] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
            vals[r[-3]] = float(r[-1].replace(",", ""))
    if "dram__bytes_read.sum" in vals:
        shutil.copy(f, os.path.join(P, os.path.basename(f)))
        key = "sh_analysis" if "k_sh" in kname else "newton_refine" if "newton" in kname else \
            "so3_search" if "so3" in kname else "corr_coeffs" if "corr" in kname else kname
        per = int(os.environ.get("PARTICLES_PER_LAUNCH", "1000"))
        warm.setdefault(key, 0.0)
        warm[key] += (vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) / per
if warm:
    out.append("DRAM traffic per particle with warm caches (ncu --cache-control none; used for roofline.traffic): " +
               ", ".join(f"{k} {v:.0f}" for k, v in warm.items()) + "\n")
    json.dump({"c2": {k: {"bytes_per_particle": v, "source": f"profiles/{tag}_warm_*.csv dram__bytes_read+write "
                                                           "(--cache-control none)"}
                      for k, v in warm.items()}}, open(os.path.join(P, "traffic.json"), "w"), indent=1)

md = os.path.join(P, f"{tag}_summary.md")
open(md, "w").write(f"# GPU evidence — {tag}\n\n" + "\n".join(out) + "\n")
print(open(md).read())
