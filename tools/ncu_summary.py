"""Summarise an ncu capture directory (tools/profile.sh output) into profiles/<round>/.

  python tools/ncu_summary.py gpurun_out/prof_r01 profiles/r01

Writes launches.md (per-kernel share of the timed region from the launch list) and
kernels.md / kernels.json (key metrics of the full-set captures)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_membar",
    "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_no_instructions",
]


def short(name):
    n = name.split("(")[0].replace("void ", "")
    for p in ["dci::(anonymous namespace)::", "(anonymous namespace)::", "<unnamed>::", "unnamed>::", "dci::"]:
        n = n.replace(p, "")
    return n


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, mi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = short(r[ki])
    agg = collections.OrderedDict()
    for i in sorted(per, key=int):
        a = agg.setdefault(names[i], [0, 0.0, 0.0, 0.0])
        m = per[i]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    return agg


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m in FULL_METRICS:
            if m in hdr:
                d[m] = r[hdr.index(m)] + ("" if not units[hdr.index(m)] else " " + units[hdr.index(m)])
        res.append(d)
    return res


def main(src, dst):
    os.makedirs(dst, exist_ok=True)
    md = ["# ncu launch list (NVTX range `timed`, serialized, cold caches: compare shares)", "",
          "| kernel | launches | avg µs | share of timed region | DRAM read MB/launch | DRAM write MB/launch |",
          "|---|---|---|---|---|---|"]
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        tot = sum(a[1] for a in agg.values())
        for k, (n, t, r, w) in agg.items():
            md.append(f"| {k} | {n} | {t / n / 1e3:.2f} | {t / tot * 100:.1f} % | {r / n / 1e6:.1f} | {w / n / 1e6:.1f} |")
        md.append("")
        md.append(f"Total kernel time in the captured steps: {tot / 1e3:.1f} µs")
    open(os.path.join(dst, "launches.md"), "w").write("\n".join(md) + "\n")
    allk = {}
    lines = ["# ncu --set full captures (key metrics)", ""]
    for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
        ks = full(os.path.join(src, rep))
        allk[rep] = ks
        lines.append(f"## {rep}")
        for k in ks:
            lines.append(f"- **{k['kernel']}**: " + ", ".join(f"{m}={v}" for m, v in k.items() if m != "kernel"))
        lines.append("")
    open(os.path.join(dst, "kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(allk, open(os.path.join(dst, "kernels.json"), "w"), indent=1)
    print("\n".join(md))
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
