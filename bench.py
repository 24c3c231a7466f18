#!/usr/bin/env python
"""DCI hot-path benchmark: seeds/s for sample+gather (BASELINE.json metric).

  python bench.py [--gpus N --steps K --warmup W] [--config M2] [--impl reference]

A step is one mini-batch through the whole hot path (S5 sample x L hops -> S6 dedup/relabel
-> S7 feature route -> S8 gather) on synthetic inputs already resident in HBM; several
steps are in flight on distinct streams/workspaces.  Setup (graph generation, S0 load,
S1 presample, S2 allocate, S3/S4 fill) happens before the timed region and is reported
as preprocessing.  Multi-GPU (torchrun, one rank per GPU): rank g runs batches g, g+G, ...
of the global list with replicated caches; presample counts are all-reduced over NCCL.

rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the reference arm
for this paper-only tier) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "seeds/s for sample+gather"
UNIT = "seeds/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="M2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--inflight", type=int, default=None,
                    help="streams in flight (each with one batch, or one group of --group batches); default 2 "
                         "groups, or 6 single batches")
    ap.add_argument("--group", type=int, default=None,
                    help="batches per dci_sample_gather_many call (one TMA gather launch per group); 0 = one "
                         "dci_sample_gather per batch.  Default (measured, DESIGN.md §9): 20 on HBM-resident data "
                         "(M1, M2), 8 on papers100M-shaped (M4, M4s), 0 on products-shaped (M3, M5)")
    ap.add_argument("--ldx", default="auto", choices=["auto", "pitch", "line"],
                    help="X row stride: the 16-byte feature pitch, or rounded up to whole 128-byte lines (the "
                         "node-sweep gather then writes whole lines: random-row writes of partial lines run ~30 %% "
                         "slower, tools/probe/scatter_probe.cu); auto = line when it adds <= 32 B per row")
    ap.add_argument("--repeats", type=int, default=5, help="timed regions of K steps (value = median)")
    ap.add_argument("--ratio", type=float, default=None, help="explicit C_adj/C split (sweeps)")
    ap.add_argument("--eq1-times", default="group", choices=["presample", "group"],
                    help="Eq. 1's T_sample / T_feature: dci_presample's per-batch stage times, or the "
                         "presample batches run as inference groups")
    ap.add_argument("--budget", default=None, help="override the config's budget (bytes:<n>|frac:<x>|auto)")
    ap.add_argument("--fanouts", default=None, help="override the config's fan-outs, e.g. 15,10,5 (DGL order)")
    ap.add_argument("--batch", type=int, default=None, help="override the config's batch size")
    ap.add_argument("--presample-batches", type=int, default=8, help="n pre-sampling batches (Fig. 11)")
    ap.add_argument("--fill", default="dci", choices=["dci", "knapsack"],
                    help="cache fill: DCI (Eq. 1 split + separate fills) or the NEXT F4 knapsack comparison")
    ap.add_argument("--cap-to-data", action="store_true",
                    help="reading B4: cap each side of the split at its data (per feature partition)")
    ap.add_argument("--partitioned", action="store_true",
                    help="NEXT F1: partition the feature cache across ranks (peer reads over NVLink)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target oracle wall time for cpu_baseline")
    ap.add_argument("--no-check", action="store_true", help="skip the bit-exact spot check vs the oracle")
    ap.add_argument("--no-latency", action="store_true", help="skip the single-batch latency measurement")
    ap.add_argument("--no-aggregate", action="store_true",
                    help="skip timing the NEXT F2 mean-aggregate consumer after the timed region")
    ap.add_argument("--check-light", action="store_true",
                    help="full-size parity without a host feature copy: oracle presample/fill/sampling on the "
                         "same graph, X rows checked against the closed-form features (papers100M-shaped)")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no baseline/check)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo only to test several ranks on one GPU)")
    ap.add_argument("--shm-graph", default="auto", choices=["auto", "on", "off"],
                    help="several ranks: one node-shared host graph adopted in place by every rank (DCI_ADOPT_HOST), "
                         "auto = when /dev/shm can hold it")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank times K batches of its shard of the global list (task rule 5: the "
                         "path shards into independent batches); strong: the K batches of one global list are "
                         "split round-robin over the ranks")
    return ap.parse_args()


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 100 ms while the region runs (every rank
    samples its own GPU, addressed by UUID so CUDA_VISIBLE_DEVICES remapping cannot mislead it)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx, self.rows, self.proc, self.th = str(gpu_index), [], None, None
        try:
            import torch
            self.idx = "GPU-" + str(torch.cuda.get_device_properties(gpu_index).uuid)
        except Exception:
            pass

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.idx)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[3:7]):
                    if v.lower().startswith("active"):
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _hostreq_table(min_bytes: int = 32, exact_bytes: int | None = None):
    """{region_GB: best GB/s over load kinds} from profiles/hostreq_probe.jsonl (tools/probe/
    hostreq_probe.cu), over request sizes >= min_bytes (or exactly exact_bytes)."""
    p = os.path.join(ROOT, "profiles", "hostreq_probe.jsonl")
    if not os.path.exists(p):
        return None
    best = {}
    for ln in open(p):
        try:
            d = json.loads(ln)
        except ValueError:
            continue
        if d.get("probe") != "host_random_read":
            continue
        if (exact_bytes is not None and d["bytes"] != exact_bytes) or d["bytes"] < min_bytes:
            continue
        best[d["region_GB"]] = max(best.get(d["region_GB"], 0.0), float(d["GBps"]))
    return sorted(best.items()) or None


def host_request_peak(region_bytes: float):
    """Best random-REQUEST rate of the host link (M requests/s) for a pinned region of this size: the
    max over request sizes (>= 32 B) and load kinds of profiles/hostreq_probe.jsonl's Mreq_per_s
    (interpolated in log2 of the region).  For regions beyond a few GB it is set by address
    translation (~70-80 M/s for 8-64 GB, whatever the size up to 512 B), not by bytes."""
    p = os.path.join(ROOT, "profiles", "hostreq_probe.jsonl")
    if not os.path.exists(p):
        return None
    best = {}
    for ln in open(p):
        try:
            d = json.loads(ln)
        except ValueError:
            continue
        if d.get("probe") == "host_random_read" and d["bytes"] >= 32:
            best[d["region_GB"]] = max(best.get(d["region_GB"], 0.0), float(d["Mreq_per_s"]))
    pts = sorted(best.items())
    return _interp_log2(pts, region_bytes / 2 ** 30) if pts else None


def _interp_log2(pts, gb):
    gb = max(gb, 1e-9)
    y = pts[0][1] if gb <= pts[0][0] else pts[-1][1]
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        if x0 <= gb <= x1:
            y = y0 + (y1 - y0) * (np.log2(gb) - np.log2(x0)) / (np.log2(x1) - np.log2(x0))
    return y


def host_link_peaks(region_bytes: float = 0.0, row_bytes: int = 512):
    """Host-link peak for the gather's miss rows: the best measured random-read rate of requests of
    the row's size (the probe's next size >= the row, e.g. 512 B for 400 B rows: an upper bound)
    for a pinned region of this size, over the probe's load kinds (profiles/hostreq_probe.jsonl;
    it falls from ~50 GB/s at 0.5-2 GB to ~35 GB/s at 64 GB for 512 B rows).  Falls back to round
    1's profiles/hostlink_peaks.json.  Returns (GB/s, random 4 B reads M/s, description)."""
    sizes = [32, 64, 128, 256, 512, 2048]
    req = next((z for z in sizes if z >= row_bytes), sizes[-1])
    tab = _hostreq_table(exact_bytes=req)
    if tab and region_bytes > 0:
        gb = region_bytes / 2 ** 30
        return (_interp_log2(tab, gb), 0.0,
                f"best measured random {req} B UVA read rate for a {gb:.1f} GB pinned region (tools/probe/hostreq_probe.cu)")
    p = os.path.join(ROOT, "profiles", "hostlink_peaks.json")
    if os.path.exists(p):
        d = json.load(open(p))
        peak, kind = float(d["uva_stream_read_GBps"]), "measured streaming UVA read (tools/probe)"
        tab = d.get("random_512B_rows_GBps_by_region_GB")
        if tab and region_bytes > 0:
            pts = sorted((float(k), float(v)) for k, v in tab.items())
            gb = region_bytes / 2 ** 30
            peak = _interp_log2(pts, gb)
            kind = f"measured random-row UVA read for a {gb:.1f} GB pinned region (tools/probe)"
        return peak, float(d["uva_random4_Mreq_per_s"]), kind
    return 51.5, 90.0, "assumed"


def host_read_peak(region_bytes: float):
    """Best random-read PAYLOAD rate of the host link (GB/s) for a pinned region of this size:
    the max over request sizes (32 B .. 2 KB) and load kinds of tools/probe/hostreq_probe.cu's
    rates (profiles/hostreq_probe.jsonl, interpolated in log2 of the region), i.e. no random read
    pattern over that region moves payload faster.  Falls back to host_link_peaks()."""
    tab = _hostreq_table(min_bytes=32)
    if not tab:
        peak, _, kind = host_link_peaks(region_bytes)
        return peak, kind
    gb = region_bytes / 2 ** 30
    return (_interp_log2(tab, gb),
            f"best random-read payload rate for a {gb:.2f} GB pinned region (tools/probe/hostreq_probe.cu)")


def _cfg(args):
    import dataclasses
    cfg = synth.CONFIGS[args.config]
    if args.fanouts:
        cfg = dataclasses.replace(cfg, fanouts=tuple(int(x) for x in args.fanouts.split(",")))
    if args.batch:
        cfg = dataclasses.replace(cfg, batch=args.batch)
    return cfg


# ------------------------------------------------------------------------------ inputs
def make_inputs(cfg, device):
    import torch
    ip_d, ix_d = synth.rmat_csc(cfg.N, cfg.E, seed=synth.GRAPH_SEED, device=device)
    ip = ip_d.cpu().numpy()
    ix = ix_d.cpu().numpy()
    del ip_d, ix_d
    ft_d = synth.features(cfg.N, cfg.D, device=device)
    ft = ft_d.cpu().numpy()
    del ft_d
    torch.cuda.empty_cache()
    return ip, ix, ft


# ------------------------------------------------------------------------------ oracle (cpu)
def light_check(cfg, ip, ix, c_adj, c_feat, gpu_results, npre=8, rows=4096):
    """Bit-exact check of GPU batches against the oracle without the feature matrix: the oracle
    presamples and fills on the same graph, samples the same seeds, and X rows are compared with
    synth.feat_fn (the closed form the features were generated from) on a random row sample."""
    import oracle
    B, fan = cfg.batch, cfg.fanouts
    pre = synth.presample_seeds(ip, npre, B)
    nv, ec = oracle.presample(ip, ix, pre, B, fan, synth.PRESAMPLE_SEED)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec, c_adj)
    del co, ac, ec
    slot, _ = oracle.feat_fill(nv, c_feat // (4 * cfg.pitch_floats()))
    ok = True
    rng = np.random.default_rng(0)
    for seeds, g in gpu_results:
        o = oracle.sample_batch(ip, R, seeds, fan, synth.SAMPLE_SEED, 0, cl)
        fh = int((slot[o.F] >= 0).sum())
        ok &= bool(np.array_equal(g["F"], o.F)
                   and all(np.array_equal(g["bsrc"][h], o.bsrc[h]) and np.array_equal(g["bptr"][h], o.bptr[h])
                           for h in range(len(fan)))
                   and g["counters"][:2].tolist() == o.counters[:2].tolist()
                   and g["counters"][2:].tolist() == [fh, len(o.F) - fh])
        idx = rng.choice(len(o.F), size=min(rows, len(o.F)), replace=False)
        ok &= bool(np.array_equal(g["X"][idx], synth.feat_fn(o.F[idx][:, None], np.arange(cfg.D)[None, :])))
    return {"batches": len(gpu_results), "bit_exact": ok,
            "mode": f"light: oracle presample+fill+sampling on the full graph, X on {rows} random rows per batch "
                    "vs the closed-form features"}


def host_mem() -> dict:
    """This process's host memory from /proc/self/status (GB): private anonymous pages, shared-memory
    pages it maps (the node-shared adopted graph counts here, once per node), and the peak RSS."""
    out = {}
    try:
        with open("/proc/self/status") as f:
            for ln in f:
                k, _, v = ln.partition(":")
                if k in ("RssAnon", "RssShmem", "RssFile", "VmHWM"):
                    out[k] = int(v.split()[0]) / 2 ** 20  # kB -> GB
    except OSError:
        pass
    return {"rss_anon_GB": out.get("RssAnon"), "rss_shmem_GB": out.get("RssShmem"),
            "rss_file_GB": out.get("RssFile"), "peak_rss_GB": out.get("VmHWM")}


def _cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_leg(cfg, ip, ix, ft, c_adj, c_feat, batches, seconds, threads, gpu_results=None, npre=8):
    """Time the oracle as it stands on host cores: its own presample + fill (reported), then
    inference batches spread over `threads` threads (ctypes releases the GIL), until about
    `seconds` of wall time.  Optionally checks the GPU results of the first batches."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    B, fan = cfg.batch, cfg.fanouts
    t0 = time.time()
    pre = synth.presample_seeds(ip, npre, B)
    nv, ec = oracle.presample(ip, ix, pre, B, fan, synth.PRESAMPLE_SEED)
    R, cl, co, ac = oracle.adj_fill(ip, ix, ec, c_adj)
    slot, _ = oracle.feat_fill(nv, c_feat // (4 * cfg.pitch_floats()))
    prep_s = time.time() - t0
    check = None
    if gpu_results:
        ok = True
        for seeds, g in gpu_results:
            o = oracle.sample_gather(ip, R, ft, seeds, fan, synth.SAMPLE_SEED, cl, slot)
            ok &= bool(np.array_equal(g["F"], o.F) and np.array_equal(g["counters"], o.counters)
                       and all(np.array_equal(g["bsrc"][h], o.bsrc[h]) and np.array_equal(g["bptr"][h], o.bptr[h])
                               for h in range(len(fan))) and np.array_equal(g["X"], o.X))
        check = {"batches": len(gpu_results), "bit_exact": ok}
    # calibrate: one batch single-threaded
    t1 = time.time()
    oracle.sample_gather(ip, R, ft, batches[0], fan, synth.SAMPLE_SEED, cl, slot)
    one = max(time.time() - t1, 1e-3)
    nb = max(threads, int(seconds * threads / one))
    nb = min(nb, 4 * threads * max(1, len(batches) // threads + 1))
    work = [batches[i % len(batches)] for i in range(nb)]
    t2 = time.time()
    def one_batch(s):
        oracle.sample_gather(ip, R, ft, s, fan, synth.SAMPLE_SEED, cl, slot)  # result dropped (memory)
        return len(s)

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(one_batch, work))
    wall = time.time() - t2
    seeds = sum(len(s) for s in work)
    return {"value": seeds / wall, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"{nb} batches of {B} seeds ({cfg.name}, {','.join(map(str, fan))}) after the oracle's own "
                      f"presample+fill ({prep_s:.1f} s, not timed); {wall:.1f} s wall on {threads} threads"}, check


def run_reference(args):
    """--impl reference: the oracle as the reference arm (rank 0 only under torchrun)."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    cfg = _cfg(args)
    import torch
    # same generator and device as our arm, so both arms see the identical graph
    gen_dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))) if torch.cuda.is_available() else "cpu"
    if gen_dev != "cpu":
        ip, ix, ft = make_inputs(cfg, gen_dev)
    else:
        ip, ix = synth.rmat_csc(cfg.N, cfg.E, seed=synth.GRAPH_SEED)
        ip, ix = ip.numpy(), ix.numpy()
        ft = synth.features(cfg.N, cfg.D).numpy()
    C = synth.parse_budget(args.budget or cfg.budget, synth.data_bytes(cfg.N, cfg.E, cfg.D))
    if C == 0:  # auto: the GPU's budget holds every byte of this workload
        C = 2 * synth.data_bytes(cfg.N, cfg.E, cfg.D)
    import oracle
    ratio = (int(round(args.ratio * 1000)), 1000) if args.ratio is not None else (1, 2)
    c_adj, c_feat = oracle.allocate(C, ratio=ratio)
    batches = synth.inference_batches(ip, cfg.batch)
    threads = os.cpu_count() or 1
    per_step = max(1, args.cpu_seconds / max(args.steps + args.warmup, 1))
    res, _ = oracle_leg(cfg, ip, ix, ft, c_adj, c_feat, batches, per_step * args.steps, threads)
    line = {"impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": cfg.batch / res["value"] * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg.name, "global_batch": cfg.batch, "fanouts": list(cfg.fanouts),
                       "N": cfg.N, "E": cfg.E, "D": cfg.D, "budget": args.budget or cfg.budget},
            "cpu_baseline": res, "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------ ours
def run_ours(args):
    import torch
    import paper_2503_01281_b200 as dci
    from paper_2503_01281_b200 import parallel

    backend = args.backend
    ndev = torch.cuda.device_count()
    if backend == "nccl" and parallel.dist_env()[1] > ndev:
        # NCCL refuses two ranks on one device: more ranks than visible GPUs run over gloo
        print(f"[bench] note: {parallel.dist_env()[1]} ranks on {ndev} visible GPU(s): gloo instead of nccl",
              file=sys.stderr)
        backend = "gloo"
    args.backend = backend
    rank, world, local = parallel.init(backend)
    if world != args.gpus:
        print(f"[bench] note: {world} ranks launched with --gpus {args.gpus}; n_gpus reports the ranks",
              file=sys.stderr)
    # one rank per GPU; (testing only) more ranks than GPUs share devices round-robin
    shared_gpus = world > torch.cuda.device_count()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = _cfg(args)
    B, fan, L = cfg.batch, cfg.fanouts, len(cfg.fanouts)
    log = (lambda *a: print(*a, file=sys.stderr, flush=True)) if rank == 0 else (lambda *a: None)
    # measured defaults: node sweeps read each feature row (HBM hit or host miss) once
    # per group -- groups of 20 on HBM-resident data (M1, M2: the driver's K = 20 is one group), of
    # 32 (DCI_MAX_GROUP) on host-resident data, where a larger group shares more miss rows (M3
    # 2.6 -> 4.7 M seeds/s, M4s 0.40 -> 1.08 M, M4 0.15 -> 0.36 M at K = 64).  A sweep probes every
    # node id in dense position tables, so papers100M-shaped M4 (whose tables would be hashed) asks
    # for dense ones: 8 N = 0.9 GB per workspace, before any is created
    default_group = {"M1": 20, "M2": 20, "M3": 32, "M4": 32, "M4s": 32, "M5": 32}.get(cfg.name.split("-")[0], 0)
    if cfg.name.startswith("M4-") and (args.group is None or args.group >= 2):
        os.environ.setdefault("DCI_TABLE", "dense")

    clk = ClockSampler(local)
    clk.start()
    # ---- inputs + S0 load.  Several ranks on one node share ONE host copy of the graph
    # (parallel.SharedGraph: local rank 0 generates it into /dev/shm, every rank's context adopts it
    # in place with DCI_ADOPT_HOST) instead of a copy per rank ----
    # (auto: with several ranks, or a single rank whose graph exceeds 16 GB -- papers100M-shaped
    # data is then pinned once, in place, instead of generated and copied into pinned memory:
    # M4 load 31 -> 11 s, peak host RSS 120 -> 69 GB; on: always)
    big = synth.data_bytes(cfg.N, cfg.E, cfg.D) > 16 * 2 ** 30
    use_shm = ((args.shm_graph == "auto" and (world > 1 or big)) or args.shm_graph == "on") and \
        parallel.SharedGraph.fits(cfg.N, cfg.E, cfg.D)
    if args.shm_graph == "on" and not use_shm:
        raise SystemExit("--shm-graph on: /dev/shm cannot hold the graph")
    t0 = time.time()
    sg = None
    if use_shm:
        def gen():
            ip_d, ix_d = synth.rmat_csc(cfg.N, cfg.E, seed=synth.GRAPH_SEED, device=dev)
            return ip_d, ix_d, synth.features(cfg.N, cfg.D, device=dev)

        sg = parallel.SharedGraph(cfg.N, cfg.E, cfg.D, gen)
        torch.cuda.empty_cache()
        ip, ix, ft = sg.indptr, sg.indices[:cfg.E], None
    else:
        ip, ix, ft = make_inputs(cfg, dev)
    t_gen = time.time() - t0
    log(f"[bench] {cfg.name}: N={cfg.N} E={cfg.E} D={cfg.D} generated in {t_gen:.1f}s"
        + (" (node-shared host graph, adopted in place)" if use_shm else ""))

    # ---- S0 load ----
    t1 = time.time()
    ctx = sg.load(local) if use_shm else dci.load_graph(ip, ix, ft, device=local)
    t_load = time.time() - t1
    if args.no_cpu_baseline or world > 1 or args.profile_only:
        ft = None  # the library holds its own pinned copy; free host RAM (papers100M-shaped: 57 GB)

    # ---- S1 presample (global list of 8 batches, sharded), C1 allreduce ----
    # (seed lists and the zeroed count arrays are harness work, outside the presample time)
    npre = args.presample_batches
    pre = synth.presample_seeds(ip, npre, B)
    pre_batches = [torch.from_numpy(pre[i * B:(i + 1) * B]).to(dev) for i in range(npre)]
    nv = torch.zeros(cfg.N, dtype=torch.int32, device=dev)
    ec = torch.zeros(cfg.E, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    ts_all, tf_all = [], []
    t2 = time.time()
    for pb in parallel.shard(pre_batches, rank, world):
        ts, tf = dci.presample(ctx, pb, B, fan, synth.PRESAMPLE_SEED, nv, ec)
        ts_all += ts.tolist()
        tf_all += tf.tolist()
    torch.cuda.synchronize()
    t_pre = time.time() - t2
    t2 = time.time()
    S, F = parallel.allreduce_presample(nv, ec, ts_all, tf_all)
    torch.cuda.synchronize()
    t_allreduce = time.time() - t2

    # ---- inference workspaces and outputs, created BEFORE the (auto) budget is cut (dci.h) ----
    G = max(0, args.group) if args.group is not None else default_group
    nws = max(1, args.inflight) if args.inflight is not None else (2 if G else 6)
    per = max(1, G)  # batches per call
    wss = [[dci.workspace_create(ctx, B, fan) for _ in range(per)] for _ in range(nws)]
    ldx_line = -(-cfg.D // 32) * 32
    line = args.ldx == "line" or (args.ldx == "auto" and 4 * (ldx_line - cfg.pitch_floats()) <= 32)
    ldx = ldx_line if line else None
    outs = [[dci.BatchOut(ctx, B, fan, ldx=ldx) for _ in range(per)] for _ in range(nws)]

    # ---- Eq. 1 inputs measured the way inference runs (--eq1-times group): the presample batches
    # once more through dci_sample_gather_many in groups (no caches yet, as in the presample), their
    # sampling / gather stage times (CUDA events) replacing the per-batch ones of dci_presample ----
    eq1_src = "presample (per batch)"
    if args.eq1_times == "group" and G >= 2 and world == 1:
        for w in wss[0]:
            w.set_profiling(True)
            w.stats(reset=True)
        torch.cuda.synchronize()
        for start in range(0, npre, per):
            chunk = pre_batches[start:start + per]
            dci.sample_gather_many(ctx, wss[0][:len(chunk)], chunk, fan, synth.PRESAMPLE_SEED, outs[0][:len(chunk)])
        torch.cuda.synchronize()
        gst = [w.stats(reset=True) for w in wss[0]]
        S = int(sum(g["sample_ms"] for g in gst) * 1e6)
        F = int(sum(g["gather_ms"] for g in gst) * 1e6)
        eq1_src = f"the presample batches as groups of {min(per, npre)} (dci_sample_gather_many stage times)"
        log(f"[bench] Eq. 1 inputs from group stage times: T_sample {S / 1e6:.2f} ms, T_feature {F / 1e6:.2f} ms")

    # ---- S2 allocate (Eq. 1) + S3/S4 fill ----
    t3 = time.time()
    C = synth.parse_budget(args.budget or cfg.budget, synth.data_bytes(cfg.N, cfg.E, cfg.D))
    ratio = (int(round(args.ratio * 1000)), 1000) if args.ratio is not None else None
    if C == 0 and world > 1:  # auto budget: the same C on every replica
        C = parallel.min_over_ranks_int(sum(dci.allocate(ctx, 0, [S], [F])), device=dev)
    c_adj, c_feat = dci.allocate(ctx, C, [S], [F], ratio=ratio)
    if args.cap_to_data:
        parts = world if (args.partitioned and world > 1) else 1
        c_adj, c_feat = parallel.cap_split_to_data(c_adj, c_feat, 4 * cfg.E, 4 * cfg.pitch_floats() * cfg.N, parts)
    if args.fill == "knapsack":
        # DUCATI-style unified budget; per-access costs profiled by the presample itself
        acc_adj = max(1, int(ec.sum(dtype=torch.int64).item()))
        acc_feat = max(1, int(nv.sum(dtype=torch.int64).item()))
        if C == 0:
            C = c_adj + c_feat
        dci.fill_knapsack(ctx, nv, ec, C, F / acc_feat, S / acc_adj)
        info0 = dci.cache_info(ctx)
        c_adj, c_feat = info0["adj_elems"] * 4, info0["feat_rows"] * 4 * info0["pitch"]
    elif args.partitioned and world > 1:
        dci.fill_partitioned(ctx, nv, ec, c_adj, c_feat, world, rank)
        torch.cuda.synchronize()
        parallel.barrier(local)
        parallel.exchange_feature_partitions(ctx)
        parallel.barrier(local)
    else:
        dci.fill(ctx, nv, ec, c_adj, c_feat)
    torch.cuda.synchronize()
    t_fill = time.time() - t3
    info = dci.cache_info(ctx)
    fill_ms = dci.fill_times(ctx)
    log(f"[bench] load {t_load:.2f}s presample {t_pre:.2f}s fill {t_fill:.2f}s  C_adj={c_adj} C_feat={c_feat} "
        f"adj_elems={info['adj_elems']}/{cfg.E} feat_rows={info['feat_rows']}/{cfg.N}")
    del nv, ec
    torch.cuda.empty_cache()

    # ---- inference batches (sharded), inputs resident in HBM ----
    batches = parallel.shard(synth.inference_batches(ip, B), rank, world)
    batches = [b for b in batches if len(b) == B] or batches
    seeds_dev = [torch.from_numpy(b).to(dev) for b in batches]
    streams = [torch.cuda.Stream(device=dev) for _ in range(nws)]
    for wl in wss:
        for w in wl:
            w.set_profiling(True)
    # exactly K timed batches (W warm-up batches): calls of `per` batches, the last one shorter if
    # K is not a multiple (the library caches both group shapes, so nothing is re-captured)
    def call_sizes(k):
        return [per] * (k // per) + ([k % per] if k % per else [])

    # weak (default): every rank times K batches; strong: the K batches of one global list are
    # split round-robin, rank g timing batches g, g+G, ... of it
    k_local = args.steps if args.scaling == "weak" else len(range(rank, args.steps, world))
    sizes = call_sizes(k_local)
    if G:
        # warm-up: at least W batches, in full groups on every stream slot, then the short last
        # shape (if any) on every slot, so both cached group graphs of each slot are the timed ones
        wsizes = [per] * max(-(-args.warmup // per), nws) + ([args.steps % per] * nws if args.steps % per else [])
    else:
        wsizes = call_sizes(args.warmup)
    n_calls = len(sizes)
    n_warm = len(wsizes)
    steps_eff = args.steps
    nxt = [0]  # rotating position in the batch list

    def take(pool, nb):
        sel = [pool[(nxt[0] + j) % len(pool)] for j in range(nb)]
        nxt[0] += nb
        return sel

    calls = {}  # (stream slot, group size) -> dci.GroupCall (workspaces, outputs, fan-outs marshalled once)

    def step(i, nb):
        w = i % nws
        if G:
            gc = calls.get((w, nb))
            if gc is None:
                gc = calls[(w, nb)] = dci.GroupCall(ctx, wss[w][:nb], fan, outs[w][:nb])
            gc(take(seeds_dev, nb), synth.SAMPLE_SEED, stream=streams[w])
        else:
            dci.sample_gather(ctx, wss[w][0], take(seeds_dev, 1)[0], fan, synth.SAMPLE_SEED, outs[w][0],
                              stream=streams[w])

    for i, nb in enumerate(wsizes):
        step(i, nb)
    torch.cuda.synchronize()
    all_ws = [w for wl in wss for w in wl]
    for w in all_ws:
        w.stats(reset=True)
    parallel.barrier(local)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream(dev)
    # the K timed steps, repeated R times (as the paper does): value = median
    R = max(1, args.repeats)
    ms_list, host_s, launches = [], 0.0, 0
    for rep in range(R):
        parallel.barrier(local)
        torch.cuda.synchronize()
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_end = torch.cuda.Event(enable_timing=True)
        launches0 = ctx.launches
        torch.cuda.nvtx.range_push("timed")
        ev_start.record(main)
        for s in streams:
            s.wait_event(ev_start)
        h0 = time.perf_counter()
        for c, nb in enumerate(sizes):
            step(n_warm + rep * n_calls + c, nb)
        host_s += time.perf_counter() - h0
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
        ev_end.record(main)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        launches += ctx.launches - launches0
        ms_local = ev_start.elapsed_time(ev_end)
        parallel.barrier(local)
        ms_list.append(parallel.max_over_ranks(ms_local, device=dev))
    ms = float(np.median(ms_list))
    ms_tot = float(np.sum(ms_list))
    host_s /= R
    launches //= R
    sts = [w.stats(reset=True) for w in all_ws]
    D = cfg.D
    rows = sum(st["frontier_rows"] for st in sts)
    cn = np.sum([st["counters"] for st in sts], axis=0).astype(np.float64)
    g_ms = sum(st["gather_ms"] for st in sts)
    s_ms = sum(st["sample_ms"] for st in sts)
    n_timed = sum(st["timed_batches"] for st in sts)
    n_glaunch = sum(st["gather_launches"] for st in sts)
    rows_read = sum(st["rows_read"] for st in sts)
    # the library's algorithmic gather bytes: row reads + row writes + lookups
    alg_bytes = float(sum(st["gather_bytes"] for st in sts))
    kinds = np.sum([st["gather_kinds"] for st in sts], axis=0)
    table_mb = max(st["table_bytes"] for st in sts) / 2 ** 20
    host_rows = sum(st["host_rows_read"] for st in sts)
    host_sectors = sum(st["host_adj_sectors"] for st in sts)
    host_runs = sum(st["host_adj_runs"] for st in sts)
    tot = parallel.sum_over_ranks([sum(st["seeds"] for st in sts), launches, rows, alg_bytes, g_ms, s_ms, n_timed,
                                   n_glaunch, rows_read, *cn.tolist(), host_rows, host_sectors, host_runs], device=dev)
    seeds_all = tot[0] / R  # per timed region
    value = seeds_all / (ms / 1e3)
    rep_values = [seeds_all / (m / 1e3) for m in ms_list]
    cn = tot[9:13]
    hit_rates = {"adj_hit_rate": cn[0] / max(1, cn[0] + cn[1]), "feat_hit_rate": cn[2] / max(1, cn[2] + cn[3]),
                 "adj_accesses_per_seed": (cn[0] + cn[1]) / max(1, tot[0])}
    if args.profile_only:
        clk.stop()
        print(json.dumps({"profile_only": True, "value": value, "ms_per_step": ms / steps_eff, **hit_rates}))
        return
    # ---- e2e: the same steps through the C-ABI with host seeds + D2H results ----
    pinned_seeds = [torch.from_numpy(b).pin_memory() for b in batches]
    e_sizes = torch.zeros((nws, per, L + 1), dtype=torch.int64).pin_memory()
    e_cnt = torch.zeros((nws, per, 4), dtype=torch.int64).pin_memory()
    e_st = torch.zeros((nws, per), dtype=torch.int32).pin_memory()
    e_res = [dci.result_buffer(per) for _ in range(nws)]
    for w in all_ws:
        w.set_profiling(False)

    def estep(i, nb):
        w = i % nws
        if G:
            gc = calls.get((w, nb))
            if gc is None:
                gc = calls[(w, nb)] = dci.GroupCall(ctx, wss[w][:nb], fan, outs[w][:nb])
            gc.host(take(pinned_seeds, nb), synth.SAMPLE_SEED, e_res[w], stream=streams[w])
        else:
            dci.sample_gather_host(ctx, wss[w][0], take(pinned_seeds, 1)[0], fan, synth.SAMPLE_SEED,
                                   outs[w][0], e_sizes[w, 0], e_cnt[w, 0], e_st[w, 0], stream=streams[w])

    for i, nb in enumerate(wsizes):
        estep(i, nb)
    torch.cuda.synchronize()
    # R timed regions of K steps, like the device-resident value above; e2e = their median
    ems_list = []
    for rep in range(R):
        parallel.barrier(local)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for s in streams:
            s.wait_event(e0)
        for c, nb in enumerate(sizes):
            estep(n_warm + rep * n_calls + c, nb)
        for s in streams:
            e = torch.cuda.Event()
            e.record(s)
            main.wait_event(e)
        e1.record(main)
        torch.cuda.synchronize()
        ems_list.append(parallel.max_over_ranks(e0.elapsed_time(e1), device=dev))
    ems = float(np.median(ems_list))
    # the same gather launch with nothing else running (3 groups, device synchronised between):
    # the kernel's own rate, next to the live per-launch rate of the pipelined timed region
    alone = None
    if G:
        for w in all_ws:
            w.stats(reset=True)
            w.set_profiling(True)
        for r in range(3):
            sd = [seeds_dev[(r * per + j) % len(seeds_dev)] for j in range(per)]
            dci.sample_gather_many(ctx, wss[0], sd, fan, synth.SAMPLE_SEED, outs[0], stream=streams[0])
            torch.cuda.synchronize()
        st0 = wss[0][0].stats(reset=True)
        if st0["gather_ms"] > 0:
            alone = {"achieved": st0["gather_bytes"] / (st0["gather_ms"] / 1e3) / 1e9,
                     "avg_gather_ms": st0["gather_ms"] / max(1, st0["gather_launches"]),
                     "launches": st0["gather_launches"]}
    # ---- batch latency (latency-bound configs report it next to seeds/s): one
    # single-batch dci_sample_gather call at a time on device-resident seeds, synchronised, CUDA
    # events on its stream; launches per batch from the library's launch counter ----
    latency = None
    if not args.no_latency:
        w0, o0 = wss[0][0], outs[0][0]
        for r in range(3):  # the single-batch shape's graph is captured here, outside the timing
            dci.sample_gather(ctx, w0, seeds_dev[r % len(seeds_dev)], fan, synth.SAMPLE_SEED, o0, stream=streams[0])
        torch.cuda.synchronize()
        lts, l0, ncall = [], ctx.launches, 20
        for r in range(ncall):
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(streams[0])
            dci.sample_gather(ctx, w0, seeds_dev[r % len(seeds_dev)], fan, synth.SAMPLE_SEED, o0, stream=streams[0])
            a1.record(streams[0])
            a1.synchronize()
            lts.append(a0.elapsed_time(a1) * 1e3)
        latency = {"us_median": float(np.median(lts)), "us_min": float(np.min(lts)), "us_max": float(np.max(lts)),
                   "launches_per_batch": (ctx.launches - l0) / ncall, "calls": ncall,
                   "note": "one single-batch dci_sample_gather at a time (B seeds on the device, nothing else "
                           "queued), after the timed regions; not part of the seeds/s value"}
    # ---- NEXT F2: the GraphSAGE mean-aggregate consumer over the input-layer block of the last
    # timed outputs (one dci_mean_aggregate launch per batch), timed alone with CUDA events ----
    consumer = None
    if not args.no_aggregate:
        agg_outs = outs[0][:per]
        torch.cuda.synchronize()
        n_dst = [int(o.sizes[L - 1].item()) for o in agg_outs]
        n_src = [int(o.sizes[L].item()) for o in agg_outs]
        n_edge = [int(o.bptr[L - 1][n_dst[i]].item()) for i, o in enumerate(agg_outs)]
        Hs = [torch.empty((max(o.bptr[L - 1].numel() - 1, 1), o.ldx), dtype=torch.float32, device=dev)
              for o in agg_outs]
        for o, Hb in zip(agg_outs, Hs):  # warm-up
            dci.mean_aggregate(ctx, o, H=Hb, stream=main)
        torch.cuda.synchronize()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        reps = 3
        a0.record(main)
        for _ in range(reps):
            for o, Hb in zip(agg_outs, Hs):
                dci.mean_aggregate(ctx, o, H=Hb, stream=main)
        a1.record(main)
        torch.cuda.synchronize()
        a_ms = a0.elapsed_time(a1) / reps
        # compulsory bytes: every source row (F_L) read once + every output row written once (+ 4 B
        # bsrc per edge, 4 B bptr per dst); edge bytes: a source row per edge (what the gather-reduce
        # requests; re-reads of a row shared by several dsts may hit L2)
        min_bytes = sum(4.0 * D * (sr + d) + 4.0 * (e + d) for sr, e, d in zip(n_src, n_edge, n_dst))
        edge_bytes = sum(4.0 * D * (e + d) + 4.0 * (e + d) for e, d in zip(n_edge, n_dst))
        hbm_pk = measured_peaks()[0]
        consumer = {"kernel": "k_mean_aggregate_v4 (dci_mean_aggregate, input-layer block, one launch per batch)",
                    "batches": len(agg_outs), "edges": sum(n_edge), "src_rows": sum(n_src), "dst_rows": sum(n_dst),
                    "ms": a_ms, "GBps": min_bytes / (a_ms / 1e3) / 1e9, "peak_GBps": hbm_pk,
                    "frac": min_bytes / (a_ms / 1e3) / 1e9 / hbm_pk,
                    "edge_GBps": edge_bytes / (a_ms / 1e3) / 1e9,
                    "note": "after the timed region (not part of the seeds/s metric); GBps = compulsory bytes "
                            "(each source row read once, each output row written once) / time; edge_GBps = a "
                            "source row per edge / time (L2 serves the re-reads)"}
    clocks = parallel.gather_clocks(clk.stop())
    clocks["window"] = "sampled every 100 ms on every rank's GPU from input generation through the e2e region"
    hm = host_mem()
    host_memory = dict(hm, max_rss_anon_GB_over_ranks=parallel.max_over_ranks(hm["rss_anon_GB"] or 0.0, device=dev),
                       note="rank 0's /proc/self/status at the end of the run; anon = private to the rank, "
                            "shmem = shared mappings: the node-shared adopted graph and the library's pinned "
                            "(cudaHostAlloc) host copies")

    e_value = seeds_all / (ems / 1e3)

    if rank != 0:
        parallel.barrier(local)
        return
    hbm_peak, peak_kind = measured_peaks()
    # Binding resource of the gather kernel: HBM (hit rows read + every row written + 4 B
    # slot lookup) vs the host link (miss rows read through UVA).
    host_peak, _, host_kind = host_link_peaks(cfg.N * 4.0 * cfg.pitch_floats(), 4 * cfg.pitch_floats())
    if kinds[0] == 0 and kinds[1] + kinds[2] > 0 and os.path.exists(os.path.join(ROOT, "profiles", "hostlink_peaks.json")):
        # every gather was a node sweep: miss rows are read in ascending node order, not at random,
        # so the link's streaming read rate bounds them (a random-request rate would be exceeded)
        host_peak = float(json.load(open(os.path.join(ROOT, "profiles", "hostlink_peaks.json")))["uva_stream_read_GBps"])
        host_kind = ("measured streaming UVA read rate (tools/probe/hostlink_probe.cu): node-sweep gathers read "
                     "the miss rows in ascending node order")
    hits_rows, miss_rows = cn[2], cn[3]
    # rows actually read: a node-sweep group reads each row once for all its batches; misses
    # among them are apportioned by the batches' miss fraction
    frac_read = tot[8] / max(1.0, tot[2])
    host_b = miss_rows * frac_read * 4.0 * D
    hbm_b = tot[3] - host_b
    host_bound = host_b / host_peak > hbm_b / hbm_peak
    bind_b = host_b if host_bound else hbm_b
    bind_peak = host_peak if host_bound else hbm_peak
    n_launch = max(1.0, tot[7])
    per_launch_gbs = bind_b / (tot[4] / 1e3) / 1e9 if tot[4] > 0 else None  # per launch (live events)
    # single-batch calls with several in flight run their gather launches concurrently, so one
    # launch's own rate says little (round-1 VERDICT): there `achieved` is the aggregate over the
    # timed wall time; group gathers run one at a time on the gather stream: per launch
    overlapped = (G == 0 and nws > 1)
    achieved_gbs = (bind_b / (ms_tot / 1e3) / 1e9) if overlapped else per_launch_gbs
    # the group gather kernels the timed regions launched (the library picks the node sweep's kernel
    # per launch: bulk copies when nothing is queued ahead of the gather, register copies otherwise)
    knames = ["k_gather_tma (rows)", "k_gather_sweep (register copies)", "k_gather_sweep_tma (bulk copies)"]
    used = {knames[i]: int(kinds[i]) for i in range(3) if kinds[i]}
    kernel = ((" + ".join(f"{k} x{v}" for k, v in used.items()) +
               f" (group of {G}; route + feature gather, S7-S8; node sweep reads each row once per group)")
              if G else "k_gather (fused route + relabel + feature gather, S7-S8)")
    aggregate_gbs = bind_b / (ms_tot / 1e3) / 1e9  # all gather launches over the timed wall time
    # Whole-step roofline of SURVEY §8(d), over all timed regions: T_roof = max(B_hbm/BW_hbm,
    # B_host/BW_host).  Algorithmic bytes: HBM = the gather's hit-row reads and all row writes
    # (+ lookups) + the sampler's cached element reads and candidate writes (4 B each); host = the
    # miss rows the gathers read (4 * pitch bytes each) + the distinct 32-byte sectors the
    # adjacency misses read (the unit the GPU fetches from system memory; the library counts both).
    # BW_host = the best random-read payload rate measured for a pinned region of the graph's size
    # (profiles/hostreq_probe.jsonl), so T_host is a lower bound on the link time of that traffic.
    host_rows_read, host_adj_sectors, host_adj_runs = tot[13], tot[14], tot[15]
    samples = cn[0] + cn[1]
    B_hbm = hbm_b + 4.0 * cn[0] + 4.0 * samples
    B_host = host_rows_read * 4.0 * cfg.pitch_floats() + 32.0 * host_adj_sectors
    region = cfg.N * 4.0 * cfg.pitch_floats() + 4.0 * cfg.E
    bw_host, bw_host_kind = host_read_peak(region)
    if kinds[0] == 0 and kinds[1] + kinds[2] > 0 and bw_host < host_peak:
        bw_host, bw_host_kind = host_peak, host_kind  # node sweeps: the streaming read rate (above)
    T_terms = {"hbm_ms": B_hbm / (hbm_peak * 1e9) * 1e3, "host_ms": B_host / (bw_host * 1e9) * 1e3}
    T_roof = max(T_terms.values())
    # Request view (SURVEY §8(d)'s N_req/R_req term, reported beside the byte roofline, not in it):
    # random host requests = miss rows + adjacency-miss runs (a run's sectors are contiguous) against
    # the best random-request rate the probe measured for a pinned region of the graph's size.  The
    # probe's requests are uniformly random, so a workload with more page locality can exceed it.
    R_req = host_request_peak(region)
    N_req = host_rows_read + host_adj_runs
    request_view = None
    if R_req and N_req > 0:
        T_req = N_req / (R_req * 1e6) * 1e3
        request_view = {"requests": N_req, "host_rows": host_rows_read, "adj_runs": host_adj_runs,
                        "M_requests_per_s": N_req / (ms_tot / 1e3) / 1e6, "peak_M_per_s": R_req,
                        "T_req_ms": T_req, "frac": T_req / ms_tot,
                        "note": "best random-request rate of tools/probe/hostreq_probe.cu for this pinned region "
                                "(address-translation bound beyond a few GB); uniformly random requests"}
    host_link = {"feature_miss_GBps": host_b / (ms_tot / 1e3) / 1e9, "peak_GBps": host_peak,
                 "feature_frac": host_b / (ms_tot / 1e3) / 1e9 / host_peak, "peak_kind": host_kind,
                 "adj_miss_Mreads_per_s": cn[1] / (ms_tot / 1e3) / 1e6,
                 "host_rows_read": host_rows_read, "host_adj_sectors": host_adj_sectors,
                 "host_payload_GBps": B_host / (ms_tot / 1e3) / 1e9, "host_read_peak_GBps": bw_host,
                 "host_read_peak_kind": bw_host_kind,
                 "request_view": request_view,
                 "step_roofline": {"T_roof_ms": T_roof, "T_measured_ms": ms_tot, "frac": T_roof / ms_tot,
                                   "binding": max(T_terms, key=T_terms.get), **T_terms,
                                   "B_hbm_bytes": B_hbm, "B_host_bytes": B_host,
                                   "note": "whole timed regions (all steps); T_roof = max(B_hbm/BW_hbm, "
                                           "B_host/BW_host), SURVEY §8(d); BW_host = best measured random-read "
                                           "payload rate for the graph's pinned region"}}
    steps_total = steps_eff * world if args.scaling == "weak" else steps_eff
    avg_fl = tot[2] / max(1, steps_total * R)
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "gather_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile)).get(f"{cfg.name}/group{G}")
        if tj:  # ncu dram bytes per launch of this kernel and configuration
            traffic = tj.get("dram_bytes_per_launch")
    # the access pattern's own measured rate (tools/probe/hbm_gather_probe.cu): context for the
    # copy-peak fraction, not a replacement for it
    pattern = None
    pfile = os.path.join(ROOT, "profiles", "hbm_pattern_peaks.json")
    if os.path.exists(pfile) and not host_bound:
        pj = json.load(open(pfile))
        wpr = 1.0 / max(frac_read, 1e-9)  # rows written per row read
        key = ("read1_write10_GBps" if wpr >= 7.5 else "read1_write5_GBps") if G and frac_read < 0.999 \
            else "gather_random_read_seq_write_GBps"
        if achieved_gbs:
            pattern = {"name": key.replace("_GBps", ""), "peak": pj[key], "frac": achieved_gbs / pj[key],
                       "writes_per_read": wpr, "source": "profiles/hbm_pattern_peaks.json"}
    # L2 rule: no flush between timed steps; say whether the inputs exceed the L2 (126 MB on B200)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    fc_mb, ac_mb = info["feat_rows"] * info["pitch"] * 4 / 1e6, info["adj_elems"] * 4 / 1e6
    x_mb = avg_fl * D * 4 / 1e6
    big = max(fc_mb, ac_mb, x_mb * min(steps_eff, per)) * 1e6 > l2_bytes
    l2_note = ("%s (L2 %.0f MB; feature cache %.0f MB, adjacency cache %.0f MB, X %.0f MB/step)"
               % ("inputs larger than L2, no flush" if big else
                  "inputs SMALLER than L2, not flushed: this config is latency-bound, not a bandwidth line",
                  l2_bytes / 1e6, fc_mb, ac_mb, x_mb))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps_eff,
        "warmup": args.warmup, "ms_per_step": ms / steps_eff, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded R-MAT graph, closed-form features)",
        "config": {"workload": cfg.name, "global_batch": B * world, "batch_per_gpu": B,
                   "ranks_share_gpus": shared_gpus, "position_table_MB_per_workspace": table_mb, "host_graph": "node-shared (adopted)" if use_shm else "per rank", "fanouts": list(fan),
                   "N": cfg.N, "E": cfg.E, "D": cfg.D, "budget": args.budget or cfg.budget,
                   "ratio": args.ratio, "fill": args.fill,
                   "parallelism": f"dp{world} (" + ("feature cache partitioned over NVLink, adjacency replicated"
                                                    if args.partitioned and world > 1 else "replicated caches") + ")",
                   "inflight": nws, "group": G, "ldx": outs[0][0].ldx, "warmup_batches_run": int(sum(wsizes)),
                   "l2": l2_note},
        "e2e": {"value": e_value, "unit": UNIT, "h2d_bytes_per_step": 4 * B,
                "d2h_bytes_per_step": (8 * dci.RESULT_WORDS) if G else (8 * (L + 1) + 8 * 4 + 4),
                "repeats": [seeds_all / (m / 1e3) for m in ems_list], "note": "median over the R timed regions"},
        "gpu_launches": int(tot[1]),
        "repeats": {"n": R, "median": value, "min": min(rep_values), "max": max(rep_values),
                    "values": rep_values, "note": "value = median seeds/s over R timed regions of K steps each"},
        "roofline": {"bound": "host-link" if host_bound else "hbm",
                     "kernel": kernel,
                     "achieved": achieved_gbs, "peak": bind_peak,
                     "achieved_kind": ("aggregate over the timed regions (overlapping single-batch gather launches)"
                                       if overlapped else "per gather launch (group gathers run one at a time)"),
                     "per_launch_achieved": per_launch_gbs,
                     "peak_kind": host_kind if host_bound else peak_kind, "unit": "GB/s",
                     "frac": (achieved_gbs / bind_peak) if achieved_gbs else None, "traffic": traffic,
                     "algorithmic_bytes_per_launch": bind_b / n_launch, "launches": int(tot[7]),
                     "avg_gather_ms": tot[4] / n_launch, "avg_sample_ms": tot[5] / max(1, tot[6]),
                     "rows_read_per_row": frac_read, "gather_kernels": used,
                     "gather_busy_frac": tot[4] / ms_tot if ms_tot > 0 else None,
                     "aggregate_achieved": aggregate_gbs, "aggregate_frac": aggregate_gbs / bind_peak,
                     "alone": None if alone is None or host_bound else dict(alone, frac=alone["achieved"] / bind_peak),
                     "pattern": pattern,
                     "note": "achieved = algorithmic bytes per gather launch / mean live launch time (CUDA events "
                             "on the launch stream) for group gathers, which run one at a time on the gather "
                             "stream; for overlapping single-batch launches the same bytes / timed wall time. "
                             "aggregate_achieved = the bytes / timed wall time; alone = the same launch "
                             "with nothing else on the GPU (3 groups after the timed region)"},
        "host_link": host_link,
        "consumer": consumer,
        "latency": latency,
        "host_memory": host_memory,
        "clocks": clocks,
        "stats": {"avg_F_L": avg_fl, "F_L_per_seed": avg_fl / B, **hit_rates,
                  "preprocess_s": {"generate": t_gen, "load": t_load, "presample": t_pre,
                                   "presample_device_s": (sum(ts_all) + sum(tf_all)) / 1e9,
                                   "presample_batches": len(ts_all), "allreduce": t_allreduce,
                                   "allocate_fill": t_fill, "fill_stages_ms": fill_ms,
                                   "note": "presample = the dci_presample calls only (seed lists and count "
                                           "arrays are made before); presample_device_s = sum of the "
                                           "per-batch CUDA-event stage times it reports (Eq. 1 inputs)"},
                  "c_adj": c_adj, "c_feat": c_feat, "eq1_times": eq1_src, "adj_elems": info["adj_elems"], "feat_rows": info["feat_rows"],
                  "e2e_ms_per_step": ems / steps_eff, "host_enqueue_ms_per_step": host_s * 1e3 / steps_eff},
    }
    def check_batches(nchk=3):
        """Full-size batches through the same call the timed region used: a whole group of `per`
        batches (the same node-sweep sampling and gather paths), of which the first `nchk` are
        checked against the oracle; or single calls."""
        if G >= 2:
            bs = [batches[j % len(batches)] for j in range(per)]
            os_ = [dci.BatchOut(ctx, B, fan) for _ in bs]
            dci.sample_gather_many(ctx, wss[0], [torch.from_numpy(b).to(dev) for b in bs], fan, synth.SAMPLE_SEED, os_)
        else:
            bs = batches[:nchk]
            os_ = [dci.BatchOut(ctx, B, fan) for _ in bs]
            for b, o in zip(bs, os_):
                dci.sample_gather(ctx, wss[0][0], torch.from_numpy(b).to(dev), fan, synth.SAMPLE_SEED, o)
        torch.cuda.synchronize()
        res = [(b, o.result()) for b, o in list(zip(bs, os_))[:nchk]]
        del os_
        return res

    if not args.profile_only and world == 1 and args.check_light:
        gpu_results = check_batches()
        line["parity_check"] = light_check(cfg, ip, ix, c_adj, c_feat, gpu_results, npre=args.presample_batches)
    if not args.profile_only and world == 1 and not args.no_cpu_baseline:
        if ft is None and sg is not None:  # single rank over the adopted shared graph
            ft = np.ascontiguousarray(sg.feats[:, :cfg.D])
        gpu_results = None
        if not args.no_check:
            gpu_results = check_batches()
        res, check = oracle_leg(cfg, ip, ix, ft, c_adj, c_feat, batches, args.cpu_seconds, os.cpu_count() or 1,
                                gpu_results, npre=args.presample_batches)
        line["cpu_baseline"] = res
        if check:
            line["parity_check"] = check
    if "parity_check" in line:
        line["parity_check"]["call"] = (f"dci_sample_gather_many, one group of {per} (as timed), first "
                                        f"{line['parity_check']['batches']} checked") if G >= 2 else "dci_sample_gather"
    print(json.dumps(line), flush=True)
    parallel.barrier(local)


def spawn_ranks(args):
    """`python bench.py --gpus N` without a torchrun environment: launch N ranks (one per GPU) through
    torch.distributed.run on this node, so the driver's plain N-GPU invocation measures N GPUs.  Rank
    0's JSON line reaches stdout; the exit code is the launcher's."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "4")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
