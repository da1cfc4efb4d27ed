"""Summarise ncu outputs (launch list CSV + one --set full report) into profiles/.

    python scripts/summarize_ncu.py <tag> <launches.csv> <full.ncu-rep> [outdir]

(outdir defaults to profiles/; gpu_ncu_round.sh summarises on the GPU box into
gpurun_out/profiles/ because the raw reports are too large to bring back.)
"""
import collections
import csv
import subprocess
import sys
from pathlib import Path

tag, launches, rep = sys.argv[1], Path(sys.argv[2]), Path(sys.argv[3])
out = Path(sys.argv[4] if len(sys.argv) > 4 else "profiles")
out.mkdir(exist_ok=True)
lines = []

rows = list(csv.reader(launches.open()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
imn = hdr.index("Metric Name")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
tot, cnt = collections.defaultdict(float), collections.Counter()
dram = collections.defaultdict(float)   # kernel family -> dram read + write bytes (all launches)


def is_ours(name: str) -> bool:   # libopara kernels live in opara::(anonymous namespace)
    return "opara::" in name or "unnamed>::" in name

ours = []
for r in data:
    name = r[ik].split("(")[0].replace("void ", "")
    metric = r[imn]
    if metric.startswith("dram__bytes_"):
        dram[name] += float(r[iv].replace(",", "")) * bscale.get(r[iu], 1)
        continue
    v = float(r[iv].replace(",", "")) * scale[r[iu]]
    tot[name] += v
    cnt[name] += 1
    if is_ours(name):
        ours.append((r[0], name, r[hdr.index("Grid Size")], r[hdr.index("Block Size")], f"{v:.3f}"))
T_ours = sum(v for k, v in tot.items() if is_ours(k))
lines.append(f"# ncu launch list — {tag}\n")
lines.append(f"Source: `{launches.name}` (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none`, cold-cache and serialised per launch: compare SHARES, "
             "not absolutes), captured inside the bench's timed region only (`--profile-region`: "
             "cudaProfilerStart/Stop around the Opara replays), so every row is a libopara kernel.\n")
lines.append("| share of our kernel time | total us | launches | DRAM MB per launch | kernel |\n|---:|---:|---:|---:|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    if is_ours(k):
        dm = f"{dram[k] / cnt[k] / 1e6:.3f}" if k in dram else "-"
        lines.append(f"| {v / T_ours * 100:5.1f}% | {v:10.1f} | {cnt[k]:5d} | {dm} | `{k}` |")
(out / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
with (out / f"{tag}_launches_ours.csv").open("w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "grid", "block", "gpu_time_us"])
    w.writerows(ours)
# per-family DRAM traffic per launch (template arguments folded: the bench's roofline names families)
fam_b, fam_n = collections.defaultdict(float), collections.Counter()
for k, v in dram.items():
    f = k.split("<")[0].split("::")[-1]
    fam_b[f] += v
    fam_n[f] += cnt[k]

# full capture
raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, u, v = rr[0], rr[1], rr[2]
d = {a: (b, c) for a, b, c in zip(h, u, v)}
keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
st = [(k, float(val[1])) for k, val in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and val[1] not in ("", "0")]
tot_s = sum(x for _, x in st) or 1
full = [f"# ncu --set full — {tag}\n", f"Source: `{rep.name}` (one launch; `--clock-control none`).\n",
        "| metric | unit | value |", "|---|---|---|"]
for k in keys:
    if k in d:
        full.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
for f in sorted(fam_b):
    full.append(f"| family dram bytes per launch: {f} | byte | {fam_b[f] / max(fam_n[f], 1):.0f} |")
full.append("\nWarp stall reasons (pc sampling):\n\n| share | reason |\n|---:|---|")
for k, x in sorted(st, key=lambda t: -t[1])[:10]:
    full.append(f"| {x / tot_s * 100:.1f}% | {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} |")
(out / f"{tag}_full.md").write_text("\n".join(full) + "\n")
print("\n".join(lines[:12]))
print("\n".join(full))
