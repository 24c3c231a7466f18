"""Sweeps over the bench (one GPU): SURVEY §8(d) M5 and NEXT F3 (Fig. 10 / Fig. 11 analogues).

  python tools/sweeps.py m5      # products-shaped, 25 % budget, r = C_adj/C in 0..1 x fan-outs
  python tools/sweeps.py budget  # products-shaped, total budget 0 .. all data (Fig. 10)
  python tools/sweeps.py npre    # products-shaped, 0.4 GB, presample batches 1..16 (Fig. 11)

Each point is one `bench.py` run (seeds/s, hit rates, Eq. 1's own split); results are appended
as JSON lines to gpurun_out/sweep_<name>.jsonl and summarised as a markdown table."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline", "--no-check", "--steps", "300", "--warmup", "10",
           "--repeats", "1"] + args
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
    if r.returncode != 0:
        return {"error": r.stderr[-500:], "args": args}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    s, h = d["stats"], d["host_link"]
    return {"args": args, "seeds_per_s": d["value"], "e2e": d["e2e"]["value"], "adj_hit": s["adj_hit_rate"],
            "feat_hit": s["feat_hit_rate"], "F_per_seed": s["F_L_per_seed"], "c_adj": s["c_adj"],
            "c_feat": s["c_feat"], "host_GBps": h["feature_miss_GBps"], "adj_miss_Mreads": h["adj_miss_Mreads_per_s"],
            "bound": d["roofline"]["bound"]}


def main(which):
    out = os.path.join(ROOT, "gpurun_out", f"sweep_{which}.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    pts = []
    if which == "m5":
        for fan in ["2,2,2", "8,4,2", "15,10,5"]:
            pts.append(["--config", "M5", "--fanouts", fan])  # Eq. 1's own split
            for r in [0.0, 0.1, 0.2, 0.3, 0.5, 0.7, 1.0]:
                pts.append(["--config", "M5", "--fanouts", fan, "--ratio", str(r)])
    elif which == "budget":
        data = 2_449_029 * 400 + 4 * 61_859_140
        for frac in [0.0, 0.05, 0.1, 0.25, 0.5, 0.75, 1.0]:
            pts.append(["--config", "M3", "--budget", f"bytes:{int(frac * data)}"])
    elif which == "npre":
        for n in [1, 2, 4, 8, 16]:
            pts.append(["--config", "M3", "--budget", "bytes:400000000", "--presample-batches", str(n)])
    rows = []
    with open(out, "a") as f:
        for a in pts:
            res = run(a)
            rows.append(res)
            f.write(json.dumps(res) + "\n")
            f.flush()
            print(json.dumps(res), flush=True)
    print("| args | seeds/s | adj hit | feat hit | C_adj MB | C_feat MB | host GB/s | adj miss M/s |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        if "error" in r:
            print(f"| {' '.join(r['args'])} | error | | | | | | |")
            continue
        print(f"| {' '.join(r['args'])} | {r['seeds_per_s'] / 1e6:.3f} M | {r['adj_hit']:.3f} | {r['feat_hit']:.3f} | "
              f"{r['c_adj'] / 1e6:.1f} | {r['c_feat'] / 1e6:.1f} | {r['host_GBps']:.1f} | {r['adj_miss_Mreads']:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])
