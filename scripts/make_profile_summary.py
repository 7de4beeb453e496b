"""Summarise an ncu capture (gpurun_out/<tag>_prof.ncu-rep + <tag>_launches.csv)
into profiles/<name>.md and profiles/<name>_launches.csv (tracked).

    python scripts/make_profile_summary.py <tag> <name> "<command that was profiled>"
"""
import csv
import io
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, name = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else ""
rep = os.path.join(ROOT, "gpurun_out", f"{tag}_prof.ncu-rep")
launches = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
out_dir = os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

M = [("gpu__time_duration.sum", "duration (us)"),
     ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
     ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
     ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
     ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
     ("smsp__inst_executed.sum", "warp instructions"),
     ("dram__bytes_read.sum", "DRAM read"),
     ("dram__bytes_write.sum", "DRAM write"),
     ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
     ("launch__registers_per_thread", "regs/thread"),
     ("launch__block_size", "block"),
     ("launch__grid_size", "grid")]

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
lines = [f"# ncu summary: {name}", "", f"Command: `{cmd}`", "",
         "Captured with `ncu --set full --clock-control none --import-source on` under gpurun "
         "(one B200, cold-cache replay; compare shares, not absolutes).", ""]
lines.append("| launch | kernel | " + " | ".join(h for _, h in M) + " |")
lines.append("|" + "---|" * (len(M) + 2))
for i, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    kname = d.get("Kernel Name", "")[:60]
    vals = []
    for key, _ in M:
        v = d.get(key, "")
        if key.startswith("dram__bytes") and v:
            v = f"{v} {u.get(key, '')}"
        if key == "gpu__time_duration.sum" and v:   # ncu picks the unit per launch
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}.get(u.get(key, ""), 1.0)
            v = f"{float(v.replace(',', '')) * scale:.3f}"
        vals.append(v)
    lines.append(f"| {i} | `{kname}` | " + " | ".join(vals) + " |")

# stall reasons per kernel and time split by code region (load / step loop / write-back)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
kernels, cur, shdr = [], None, None
for r in csv.reader(io.StringIO(src)):
    if r and r[0] == "Kernel Name":
        cur = []
        kernels.append(cur)
        continue
    if r and r[0] == "Address":
        shdr = r
        continue
    if cur is not None and len(r) > 5:
        cur.append(r)
nk = len(rows) - 2
if nk and len(kernels) == 2 * nk:   # the source page lists each kernel twice
    kernels = kernels[::2]
lines += ["", "## Warp-stall samples by region and top stall reasons", "",
          "Regions: `load` = before the first VOTE of the step loop, `loop` = step loop, "
          "`post` = write-back/compaction.", "",
          "| launch | load | loop | post | top stall reasons (share of samples) |", "|---|---|---|---|---|"]
for i, k in enumerate(kernels):
    seen, reg, stalls = 0, {"load": 0, "loop": 0, "post": 0}, {}
    for r in k:
        d = dict(zip(shdr, r))
        s = int(d.get("Warp Stall Sampling (All Samples)") or 0)
        if "VOTE.ANY P" in d.get("Source", ""):
            seen += 1
        reg["load" if seen == 0 else ("loop" if seen <= 2 else "post")] += s
        for kk in shdr:
            if kk.startswith("stall_") and "(Not" not in kk:
                stalls[kk] = stalls.get(kk, 0) + int(d.get(kk) or 0)
    tot = sum(reg.values()) or 1
    top = ", ".join(f"{a[6:]} {b / tot:.2f}" for a, b in sorted(stalls.items(), key=lambda x: -x[1])[:5])
    lines.append(f"| {i} | {reg['load'] / tot:.2f} | {reg['loop'] / tot:.2f} | {reg['post'] / tot:.2f} | {top} |")

with open(os.path.join(out_dir, f"{name}.md"), "w") as f:
    f.write("\n".join(lines) + "\n")
if os.path.exists(launches):
    shutil.copy(launches, os.path.join(out_dir, f"{name}_launches.csv"))
print(os.path.join(out_dir, f"{name}.md"))
