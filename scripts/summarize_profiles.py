"""Turns gpurun_out/ ncu artefacts into the tracked summaries under profiles/ (run here, no GPU needed).
usage: python scripts/summarize_profiles.py <profiles-tag> [gpurun_out-tag] [bench args as text]"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict, defaultdict

tag = sys.argv[1]
variant = sys.argv[2] if len(sys.argv) > 2 else "v0"
bench_args = sys.argv[3] if len(sys.argv) > 3 else ""
os.makedirs("profiles", exist_ok=True)

# ---- launch list: per-kernel share of the step ----------------------------------------------------------
src = f"gpurun_out/launches_{variant}.csv"
rows = []
with open(src) as f:
    lines = [l for l in f if not l.startswith("==")]
rd = csv.reader(io.StringIO("".join(lines)))
hdr = next(rd)
ix = {h: i for i, h in enumerate(hdr)}
for r in rd:
    if len(r) < len(hdr):
        continue
    rows.append((int(r[ix["ID"]]), r[ix["Kernel Name"]], float(r[ix["Metric Value"]]), r[ix["Metric Unit"]]))
unit = rows[0][3]
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "usecond": 1.0, "nsecond": 1e-3}.get(unit, 1.0)


def short(name):
    if "pair_kernel" in name:
        args = name[name.index("<") + 1: name.index(">")].replace(" ", "").split(",")
        mode = {"0": "fwd", "1": "adj", "2": "vel"}[args[2]]
        return f"pair_kernel<{args[0]},D{args[1]},{mode},R{args[3]},JU{args[4]},minb{args[5]}{',f32x2' if len(args) > 6 and args[6] in ('1','true') else ''}>"
    return name.split("(")[0].split("<")[0]


# one evaluation = the last 2T+2(+memset) launches before the end; find the last aos_to_planes and take from there
names = [short(n) for _, n, _, _ in rows]
last = max(i for i, n in enumerate(names) if "aos_to_planes" in n)
prev = max(i for i, n in enumerate(names[:last]) if "aos_to_planes" in n)
step = [r for r in rows[prev:last] if 'at::' not in r[1]]  # torch's L2-flush fill sits between evaluations
tot = sum(r[2] for r in step) * scale
agg = OrderedDict()
for _, n, v, _ in step:
    k = short(n)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v * scale
shutil.copy(src, f"profiles/{tag}_launches.csv")
with open(f"profiles/{tag}_launches.md", "w") as f:
    f.write(f"# {tag}: ncu launch list of `python bench.py --steps 2 --warmup 3 --no-extras {bench_args}`\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (cold-cache, serialised: compare SHARES).\n")
    f.write(f"Raw list: `profiles/{tag}_launches.csv`.  One objective evaluation (launches {rows[prev][0]}..{rows[last-1][0]}):\n\n")
    f.write("| kernel | launches | total us | avg us | share of step |\n|---|---:|---:|---:|---:|\n")
    for k, (c, t) in agg.items():
        f.write(f"| `{k}` | {c} | {t:.1f} | {t/c:.1f} | {100*t/tot:.1f} % |\n")
    f.write(f"| **step** | {len(step)} | {tot:.1f} | | 100 % |\n")
print(open(f"profiles/{tag}_launches.md").read())

# ---- full capture: the counters the roofline discussion uses ---------------------------------------------------
rep = f"gpurun_out/prof_{variant}.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rd = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rd[0], rd[1], rd[2:]
ix = {h: i for i, h in enumerate(hdr)}
keep = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_static", "launch__occupancy_limit_registers", "sm__cycles_elapsed.max",
    "sm__cycles_active.avg", "sm__cycles_active.min", "sm__cycles_active.max",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]
with open(f"profiles/{tag}_ncu_full.md", "w") as f:
    f.write(f"# {tag}: `ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 49 -c 2` "
            f"on `python bench.py --steps 1 --warmup 3 --no-extras {bench_args}`\n\n")
    f.write("The last forward and the first adjoint pair-kernel launch of a warm-up evaluation (N = 20 000, T = 10).\n\n")
    f.write("| metric | unit | " + " | ".join(short(d[ix["Kernel Name"]]) for d in data) + " |\n")
    f.write("|---|---|" + "---:|" * len(data) + "\n")
    for k in keep:
        if k in ix:
            f.write(f"| `{k}` | {units[ix[k]]} | " + " | ".join(d[ix[k]] for d in data) + " |\n")
print(open(f"profiles/{tag}_ncu_full.md").read()[:3000])

# ---- DRAM traffic per launch of the dominant kernels (bench.py's roofline.traffic) ----------------------------------
def kb(v, u):
    return float(v) * {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)


traffic = {}
for d in data:
    name = short(d[ix["Kernel Name"]])
    rd_b = kb(d[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
    wr_b = kb(d[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
    traffic.setdefault(name, []).append(rd_b + wr_b)
out = {"source": f"profiles/{tag}_ncu_full.md (dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full)",
       "kernels": {k: sum(v) / len(v) for k, v in traffic.items()}}
json.dump(out, open(f"profiles/{tag}_traffic.json", "w"), indent=1)
print(out)
