"""Summarise ncu reports into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out_prefix>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, launches, prefix = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size"]
out = {}
md = ["| kernel | metric | value | unit |", "|---|---|---|---|"]
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    d = {}
    for k in keys:
        if k in hdr:
            d[k] = (r[hdr.index(k)], units[hdr.index(k)])
            md.append(f"| {name[:60]} | {k} | {d[k][0]} | {d[k][1]} |")
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    d["top_stalls"] = stalls[:6]
    md.append(f"| {name[:60]} | top stalls (warps per issue) | {stalls[:6]} | |")
    out[name] = d


def gb(x, unit):
    v = float(x.replace(",", ""))
    return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(unit, 1.0)


traffic = {}
# the primal step = every kernel mq_primal_step launches (one launch each in
# the capture): screened solve + full-solve list + medium / long rows, or the
# unscreened tile kernel
PRIMAL = ("ws_kernel", "ws_full_kernel", "primal_med", "primal_long", "primal_fused")
rd = wr = 0.0
names = []
for name, d in out.items():
    if any(t in name for t in PRIMAL):
        rd += gb(*d["dram__bytes_read.sum"])
        wr += gb(*d["dram__bytes_write.sum"])
        names.append(name.split("(")[0])
if names:
    traffic["primal"] = {"dram_bytes_per_launch": (rd + wr) * 1e9, "read_gb": rd,
                         "write_gb": wr, "kernels": names, "source": rep,
                         "config": "c4"}
json.dump(traffic, open("profiles/ncu_traffic.json", "w"), indent=1)
# launch list: per-kernel share of device time
tot = defaultdict(float)
cnt = defaultdict(int)
with open(launches) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
rdr = csv.reader(io.StringIO("".join(lines)))
lh = next(rdr)
for r in rdr:
    if len(r) < len(lh):
        continue
    rec = dict(zip(lh, r))
    if rec.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(rec["Metric Value"].replace(",", ""))
    unit = rec.get("Metric Unit", "nsecond")
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
    k = rec["Kernel Name"].split("(")[0][:70]
    tot[k] += v
    cnt[k] += 1
S = sum(tot.values())
md += ["", "## Launch list (ncu, cold-cache, serialised)", "", "| kernel | launches | total ms | share |",
       "|---|---|---|---|"]
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    md.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / S:.1f}% |")
ITER = ("primal_fused", "ws_kernel", "ws_full_kernel", "dual_kernel", "colsum_finalize",
        "chunk_end", "primal_long", "primal_med", "cs_from_fixed", "avg_materialize")
it = {k: v for k, v in tot.items() if any(t in k for t in ITER)}
SI = sum(it.values()) or 1.0
md += ["", "## Per-iteration kernels only (the bench's timed region)", "",
       "| kernel | launches | total ms | share of iteration |", "|---|---|---|---|"]
for k, v in sorted(it.items(), key=lambda kv: -kv[1]):
    md.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / SI:.2f}% |")
open(prefix + ".md", "w").write("\n".join(md) + "\n")
print("\n".join(md[-12:]))
