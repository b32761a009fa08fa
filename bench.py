#!/usr/bin/env python
"""Benchmark: words/sec of the HogBatch SGNS step on BASELINE.json cfg3 (V=1M, D=300, 800M
planted Zipf(1.07) tokens, window=5, K=5, t=1e-4), 1..8 B200s, plus its rooflines.

A step = one `w2v_train(corpus, n, 1)` call = every SURVEY.md §8(a) row over the whole corpus
(setup a0, subsampling/window a1, sampler a2, fused step a3-a7, L2 hints a8, and with N>1 the
model averaging a9 every 2^20 words per GPU). `value` is device-timed (CUDA events on the
library's stream, max over ranks) with the corpus resident in HBM; `e2e` is the same call with a
pinned HOST corpus (H2D inside the timed region). `--impl reference` times the CPU oracle.

Rooflines, every denominator measured in this run except HBM's:
  roofline       the BINDING resource, the L2 row path: algorithmic row bytes B_row of the timed
                 calls / step-kernel time, against the in-run cap of the same access pattern
                 (tools/peaks.cu peaks_l2_rowpath: bulk gather + bulk reduce of the model's rows,
                 L2-resident, all SMs);
  roofline_hbm   BASELINE.json's "fraction of gather/scatter HBM roofline": the same B_row rate
                 against the measured HBM copy bandwidth (MEASURED_PEAKS.json). It exceeds 1
                 because L2 serves the Zipf-hot rows; DRAM bytes actually moved are in `traffic`;
  roofline_cache the survey's cache-aware bound T_roof = max(B_row/BW_L2, B_cold/BW_HBM,
                 FLOP/FMA_peak) over the measured step-kernel time;
  fma            the FMA-pipe share: 6·D·loss_pairs FLOP / step-kernel time vs the in-run FFMA2
                 peak (tools/peaks.cu peaks_ffma2).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import platform
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import inputs  # noqa: E402

METRIC = "words/sec (1/2/4/8 B200) and fraction of gather/scatter HBM roofline"
CFG = 3
WORKLOADS = {
    3: "cfg3: V=1,000,000 D=300 window=5 K=5 t=1e-4 alpha=0.025, 800M planted Zipf(1.07) tokens "
       "(C=10,000, L=20), 1 epoch per step",
    4: "cfg4: V=1,000,000 D=128 window=8 K=15 t=1e-5 alpha=0.025, 800M iid Zipf(1.07) tokens (L=1000), "
       "1 epoch per step",
    5: "cfg5: V=4,000,000 D=300 window=5 K=5 t=1e-4 alpha=0.025, 8B iid Zipf(1.05) tokens generated "
       "on-device (L=1000), 1 epoch per step",
}
SYNC_P = 1 << 20
REF_SAMPLE = 1 << 17      # raw words per thread per reference step (bounded CPU sample of cfg3)
BASE_SAMPLE = 1 << 19     # raw words per thread for the cpu_baseline leg
PEAKS_SO = os.path.join(ROOT, "tools", "libw2v_peaks.so")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload_config(args, world: int) -> dict:
    """The `config` object of BOTH arms (ours and --impl reference): the workload, not the run."""
    cfg = inputs.CONFIGS[args.config]
    n = args.tokens if args.tokens else cfg.n
    hot, cold = sync_scheme(args, cfg, world)
    return {"workload": WORKLOADS[args.config], "V": cfg.V, "D": cfg.D, "window": cfg.window, "K": cfg.K,
            "t": cfg.t, "n_tokens": n, "full_size": n == cfg.n, "epochs_per_step": 1,
            "sync_period_words": args.sync_period if world > 1 else None,
            "sync": sync_name(hot, cold, args.sync_overlap > 0) if world > 1 else None,
            "parallelism": f"dp{world} corpus-sharded replicas" if world > 1 else "single GPU",
            "l2": "no flush: corpus (3.2 GB) and model (2.4 GB) exceed the 126 MB L2" if args.config != 5 else
                  "no flush: corpus (32 GB) and model (9.6 GB) exceed the 126 MB L2",
            "algorithm": "hogbatch" if args.algorithm == "hogbatch" else "alg1 (PAPER.md:37-63, level-1 baseline)"}


def sync_scheme(args, cfg, world):
    """C13 (the paper's protocol, BASELINE cfg3: full-model average every 2^20 words per GPU) is
    the default; C14 hot/cold is opt-in (--sync-hot-rows H --sync-cold-every C)."""
    hot = max(args.sync_hot_rows, 0) if world > 1 else 0
    cold = max(args.sync_cold_every, 1) if world > 1 else 1
    return hot, cold


def sync_name(hot, cold, ovl):
    s = ("C13: full-model allreduce average (ncclAvg) after every interval" if hot == 0 or cold <= 1 else
         f"C14: rows [0,{hot}) averaged every interval, the rest every {cold}th and at the end")
    if ovl:
        s += "; C15: each average in flight (out-of-place) during the next interval, applied one interval late"
    return s


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 7 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 7 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 7 for i in range(4) if r[4 + i] == "Active"})
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        pw = [num(r[8]) for r in self.rows if len(r) > 9 and num(r[8]) is not None]
        lim = [num(r[9]) for r in self.rows if len(r) > 9 and num(r[9]) is not None]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w": float(np.median(pw)) if pw else None, "power_limit_w": max(lim) if lim else None}


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _oracle_time(cfg, n, threads, prec, reps=1, warm=0):
    """Seconds for `reps` Hogwild-threaded oracle passes over the first n raw words of cfg (setup
    excluded; a fresh contract-init model; threads = 1 runs the sequential O-HB)."""
    import oracle
    ids = cfg.corpus().tokens(0, n)
    c = oracle.counts(ids, cfg.V)
    thr, P = oracle.thresholds(c, n, cfg.t), oracle.sampler(c)
    prm = oracle.make_params(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed, cfg.L, 1, n)
    mi, mo = oracle.init(cfg.V, cfg.D, cfg.seed)
    dt = oracle.real_dtype(prec)
    M_in, M_out = mi.astype(dt), mo.astype(dt)
    del mi, mo
    nch = (n + cfg.L - 1) // cfg.L
    for _ in range(warm):
        oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), threads, prec)
    t0 = time.perf_counter()
    for _ in range(reps):
        if threads == 1:
            oracle.train_range(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), None, prec)
        else:
            oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), threads,
                                       prec)
    return time.perf_counter() - t0


def cpu_baseline(cfg, sample):
    """The oracle on the box's host cores: its Hogwild threaded mode
    ("parallelized over threads without any additional change") over all host
    threads, fp32 (the GPU path's precision) built -O3 -march=native for this host; plus the
    same in fp64 (-O2, the parity build) and the sequential fp64 O-HB on one core. Setup excluded.
    A deliberately simple program: the GPU/CPU ratio says nothing about kernel quality."""
    import oracle
    T = host_threads()
    flags = oracle.build_native()
    n = sample * T
    dt32 = _oracle_time(cfg, n, T, "f32native")
    dt64 = _oracle_time(cfg, n, T, "f64")
    dt1 = _oracle_time(cfg, sample, 1, "f64")
    return {"value": n / dt32, "unit": "words/s", "cores": T, "kind": "oracle",
            "sample": f"first {n} raw words of cfg{cfg.idx} (V={cfg.V}, D={cfg.D}), fp32 O-HB in the oracle's "
                      f"Hogwild threaded mode on {T} host threads, setup excluded",
            "seconds": dt32, "cpu_model": cpu_model(), "nproc": os.cpu_count(), "threads": T,
            "compiler": f"gcc {flags}",
            "value_fp64": n / dt64, "compiler_fp64": "gcc " + " ".join(oracle.CFLAGS) + " -DREAL=double",
            "value_1core": sample / dt1,
            "sample_1core": f"first {sample} raw words, sequential fp64 O-HB, 1 thread ({dt1:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = inputs.CONFIGS[args.config]
    import oracle
    T = host_threads()
    flags = oracle.build_native()
    n = REF_SAMPLE * T
    dt = _oracle_time(cfg, n, T, "f32native", reps=args.steps, warm=args.warmup)
    v = n * args.steps / dt
    sample = (f"first {n} raw words of cfg{cfg.idx} per step (a bounded sample of the workload), fp32 oracle "
              f"(O-HB) in its Hogwild threaded mode on {T} host threads, gcc {flags}")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "words/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": v, "unit": "words/s", "cores": T, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": v, "unit": "words/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    return 0


def measure_caps(row_bytes, rows_per_target, units_per_sm):
    """In-run roofline denominators (tools/peaks.cu): the L2 row-path cap of this access pattern
    (max over a few residencies, R = rows per target) and the FFMA2 peak. None if unavailable."""
    if not os.path.exists(PEAKS_SO):
        return None
    lib = ctypes.CDLL(PEAKS_SO)
    d = ctypes.c_double(0.0)
    mhz = ctypes.c_double(0.0)
    caps, clk = {}, {}
    for w in sorted({units_per_sm, 8, 12, 16}):
        if lib.peaks_l2_rowpath_clk(int(row_bytes), int(rows_per_target), int(w), 0, ctypes.byref(d),
                                    ctypes.byref(mhz)) == 0:
            caps[w], clk[w] = d.value, mhz.value
    best = max(caps, key=caps.get) if caps else None
    # the SM clock each cap run ran at (clock64 over its event time)
    out = {"l2_rowpath_gbs": caps[best] if caps else None, "l2_rowpath_by_units": caps,
           "l2_rowpath_sm_mhz": clk.get(best), "l2_rowpath_sm_mhz_by_units": clk}
    if lib.peaks_ffma2(ctypes.byref(d)) == 0:
        out["ffma2_tflops"] = d.value
    if lib.peaks_l2_read(ctypes.byref(d)) == 0:
        out["l2_read_gbs"] = d.value
    if lib.peaks_l2_red(ctypes.byref(d)) == 0:
        out["l2_red_gbs"] = d.value
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1611_06172_b200 import binding as w2v

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # communicator lines (nRanks) for the driver's log
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = inputs.CONFIGS[args.config]
    n = args.tokens if args.tokens else cfg.n      # --tokens: profiling only (prefix of the config)
    start, end = w2v.dist_shard(n, cfg.L, world, rank)
    n_local = end - start
    # the shard is generated on the device (inputs/gen_cuda.cu, bit-identical to the host
    # generator; cfg5 is "generated on-device from seed") and copied once to pinned host memory
    # for the e2e leg
    dev = torch.empty(max(n_local, 1), dtype=torch.int32, device="cuda")
    cfg.corpus().tokens_cuda(start, n_local, dev)
    host = torch.empty(max(n_local, 1), dtype=torch.int32, pin_memory=True)
    host.copy_(dev)
    torch.cuda.synchronize()

    w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
    w2v.set_option("sentence_len", cfg.L)
    w2v.set_option("sync_period_words", args.sync_period)
    hot, cold = sync_scheme(args, cfg, world)
    w2v.set_option("sync_hot_rows", hot)      # 0 = C13 full averaging (default)
    w2v.set_option("sync_cold_every", cold)
    ovl = int(args.sync_overlap > 0)
    w2v.set_option("sync_overlap", ovl)
    w2v.set_option("sync_device", int(args.sync_device > 0))   # C17: must precede dist_init
    w2v.set_option("kernel", args.kernel)
    if args.scatter_wait >= 0:
        w2v.set_option("scatter_wait", args.scatter_wait)
    w2v.set_option("algorithm", 1 if args.algorithm == "alg1" else 0)
    stream = torch.cuda.current_stream()
    w2v.set_stream(stream.cuda_stream)
    if world > 1:
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(w2v.dist_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        w2v.dist_init(rank, world, bytes(uid.cpu().numpy().tolist()))
    else:
        w2v.dist_init(0, 1, None)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def maxr(*vals):
        t = torch.tensor(vals, dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t]

    for _ in range(args.warmup):
        w2v.train(dev, n_local, 1)
    barrier()
    steps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    before = w2v.get_stats()
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            w2v.train(dev, n_local, 1)
            steps.append(w2v.get_stats())
        e1.record(stream)
        barrier()
    # counters (words, targets, row_touches, loss_pairs, loss_sum) are cumulative since w2v_init:
    # the last timed call's own values are differences
    prev = steps[-2] if len(steps) > 1 else before
    call = {k: steps[-1][k] - prev[k] for k in ("words", "targets", "row_touches", "loss_pairs", "loss_sum")}
    ms = e0.elapsed_time(e1)
    ms_step_kernel = sum(s["ms_step"] for s in steps) / len(steps)
    ms_max, kern_max = maxr(ms, ms_step_kernel)
    value = n * args.steps / (ms_max / 1e3)

    # e2e: the same call, every timed step, with a pinned HOST corpus and the step's statistics
    # (loss) read back to the host. Every step's corpus crosses PCIe inside the timed region:
    # step 0's before it trains, step s+1's on the copy engine (w2v_prefetch) while step s trains
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    w2v.prefetch(host, n_local)
    for s in range(args.steps):
        if s + 1 < args.steps:
            w2v.prefetch(host, n_local)
        w2v.train(host, n_local, 1)
        w2v.get_stats()
    f1.record(stream)
    barrier()
    te, = maxr(f0.elapsed_time(f1))
    e2e_value = n * args.steps / (te / 1e3)
    last = steps[-1]

    # row-path roof: the same kernel and batch stream with a4-a6 skipped (zero deltas reduced,
    # model unchanged) — what the gathers + scatters alone sustain on this chip
    roof = None
    if args.algorithm == "hogbatch" and args.kernel in (0, 1, 4) and not args.no_rowpath:
        w2v.set_option("rowpath_only", 1)
        w2v.train(dev, n_local, 1)
        rs = w2v.get_stats()
        w2v.set_option("rowpath_only", 0)
        tr, = maxr(rs["ms_step"])
        roof = n / (tr / 1e3)

    if rank == 0:
        peak, peak_src = peaks()
        kern_s = last["ms_step"] / 1e3
        bps = last["bytes_row"] / kern_s                       # algorithmic row bytes / s
        rows_per_target = call["row_touches"] / max(call["targets"], 1)
        caps = measure_caps(4 * cfg.D, max(1, round(rows_per_target)), last["units_per_sm"])
        traffic = None   # DRAM bytes per launch (ncu --set full capture, profiles/), scaled to this launch size
        traffic_src = None
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof) and args.algorithm == "hogbatch":
            tr = json.load(open(prof))
            if tr.get("config", 3) == args.config and tr.get("kernel_id", last["kernel"]) == last["kernel"]:
                traffic = tr.get("dram_bytes_per_word") * n_local / max(last["step_launches"], 1)
                traffic_src = f"ncu --set full capture {tr.get('source')} ({tr.get('round')}), profiles/ncu_traffic.json"
        flop = 6.0 * cfg.D * call["loss_pairs"]                 # 3 FMA per (pair, column): a4, a6 (x2)
        out = {
            "metric": METRIC, "value": value, "unit": "words/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args, world),
            "run": {"units_per_sm": last["units_per_sm"], "mode": "hogwild",
                    "kernel": {1: "rows", 2: "window", 3: "window-wg", 4: "alg1", 5: "ring"}.get(last["kernel"]),
                    "step_launches_per_step": last["step_launches"],
                    "sync_path": {0: None, 1: "nccl allreduce (ncclAvg)",
                                  2: "C17 device kernel, NVLink peer loads/stores",
                                  3: "C17 device kernel, NVLS multimem"}.get(last["sync_path"])},
            # per call the library reads back its setup info (32 B) before training and its
            # statistics (72 B) + finite-check flag block (32 B) after it
            "e2e": {"value": e2e_value, "unit": "words/s", "h2d_bytes_per_step": n_local * 4,
                    "d2h_bytes_per_step": 32 + 72 + 32, "steps": args.steps,
                    "h2d": "pinned host corpus; step 0 copied before it trains, step s+1 copied on the copy "
                           "engine (w2v_prefetch) while step s trains"},
            "gpu_launches": int(sum(s["launches"] for s in steps)),
            "clocks": clk.summary(),
        }
        clk_summary = out["clocks"]
        l2cap = caps and caps.get("l2_rowpath_gbs")
        if l2cap:
            out["roofline"] = {
                "bound": "l2", "achieved": bps / 1e9, "peak": l2cap, "unit": "GB/s", "frac": bps / 1e9 / l2cap,
                "traffic": traffic, "kernel": "hogbatch_step" if args.algorithm == "hogbatch" else "alg1",
                "what": "algorithmic row bytes B_row = row_touches x 4D x 2 (gather + scatter) per launch / "
                        "step-kernel time; peak = in-run cap of the same access pattern (tools/peaks.cu "
                        f"peaks_l2_rowpath: bulk gather + bulk reduce of {4 * cfg.D}-B rows, "
                        f"{max(1, round(rows_per_target))} rows per batch, L2-resident, all SMs)",
                "traffic_source": traffic_src,
                # bytes the kernel really moved through L2 (fewer than B_row for the ring kernel,
                # which keeps a chunk's M_in window on chip) and that rate against the same cap
                "moved_gbs": last["bytes_moved"] / kern_s / 1e9,
                "moved_frac": last["bytes_moved"] / kern_s / 1e9 / l2cap,
                "algorithmic_bytes_per_launch": last["bytes_row"] / max(last["step_launches"], 1),
                "kernel_ms_per_step": kern_max, "kernel_share_of_step": kern_max / (ms_max / args.steps)}
            # context: the SM clock the best cap run ran at (clock64 over its event time) beside
            # the timed region's (clocks.sm_mhz); the cap's bytes/s barely move with the SM clock
            # (L2 has its own), the kernel's follow it (its issue/latency side), r02_ablations §19
            out["roofline"]["cap_sm_mhz"] = caps.get("l2_rowpath_sm_mhz")
            out["roofline"]["run_sm_mhz"] = (clk_summary or {}).get("sm_mhz")
        else:  # tools lib missing: report against HBM only
            out["roofline"] = {"bound": "hbm", "achieved": bps / 1e9, "peak": peak, "unit": "GB/s",
                               "frac": bps / 1e9 / peak, "traffic": traffic}
        out["roofline_hbm"] = {
            "bound": "hbm", "achieved": bps / 1e9, "peak": peak, "unit": "GB/s", "frac": bps / 1e9 / peak,
            "peak_source": peak_src, "row_bytes_per_word": last["bytes_row"] / n_local,
            "what": "BASELINE.json's gather/scatter HBM roofline fraction (R_HBM, SURVEY.md §8(d)): B_row rate / "
                    "HBM copy bandwidth; > 1 because L2 serves the Zipf-hot rows",
            "dram_frac": None if traffic is None else traffic * max(last["step_launches"], 1) / kern_s / 1e9 / peak}
        if caps:
            bcold = last["row_touches_cold"] * 4 * cfg.D * 2
            t_roof = max(last["bytes_row"] / (l2cap * 1e9) if l2cap else 0.0, bcold / (peak * 1e9),
                         flop / (caps.get("ffma2_tflops", 1e9) * 1e12))
            out["roofline_cache"] = {
                "frac": t_roof / kern_s, "t_roof_ms": t_roof * 1e3, "t_meas_ms": kern_s * 1e3,
                "b_row": last["bytes_row"], "b_cold": bcold, "cold_from_row": last["cold_from_row"],
                "what": "T_roof = max(B_row / L2 row-path cap, B_cold / HBM, FLOP / FFMA2 peak) over the step-kernel "
                        "time (SURVEY.md §8(d)); B_cold = touches of rows outside the L2-sized hot prefix x 4D x 2"}
            out["fma"] = {"achieved_tflops": flop / kern_s / 1e12, "peak_tflops": caps.get("ffma2_tflops"),
                          "frac": flop / kern_s / 1e12 / caps["ffma2_tflops"] if caps.get("ffma2_tflops") else None,
                          "what": "6 D FLOP per (input, output) pair (a4 dots, a6 both updates) / step-kernel time vs "
                                  "the in-run FFMA2 peak (tools/peaks.cu peaks_ffma2)"}
            out["caps"] = caps
        if roof is not None:
            out["rowpath_roof"] = {
                "value": roof, "unit": "words/s", "frac": (n / (kern_max / 1e3)) / roof,
                "how": "same step kernel, launch configuration and batch stream with a4-a6 skipped (zero "
                       "deltas reduced): the gather/scatter path alone; frac = step-kernel words/s / roof"}
        out["stats"] = {"loss_per_pair": call["loss_sum"] / max(call["loss_pairs"], 1),
                        "ms_setup": last["ms_setup"], "ms_step": last["ms_step"], "ms_batch": last["ms_batch"],
                        "ms_sync": last["ms_sync"], "syncs": last["syncs"], "syncs_hot": last["syncs_hot"],
                        "targets_per_word": call["targets"] / n_local, "rows_per_target": rows_per_target,
                        "bytes_moved_per_word": last["bytes_moved"] / n_local}
        if world == 1 and not args.no_cpu_baseline and cfg.V * cfg.D <= 300_000_000:
            out["cpu_baseline"] = cpu_baseline(cfg, BASE_SAMPLE)
        elif world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = {"value": None, "unit": "words/s", "cores": 1, "kind": "oracle",
                                   "sample": "skipped: the fp64 oracle model (2*V*D*8 bytes) exceeds the host budget"}
        print(json.dumps(out))
    w2v.finalize()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-rowpath", action="store_true", help="skip the rowpath_only roof run")
    ap.add_argument("--kernel", type=int, default=0,
                    help="0 auto, 1 per-target rows, 2 window-resident rows, 3 window-resident warp-specialised, "
                         "4 ring (window-resident M_in rows, originals in TMEM)")
    ap.add_argument("--tokens", type=int, default=0, help="profiling only: train on a prefix of the config")
    ap.add_argument("--config", type=int, choices=[3, 4, 5], default=CFG,
                    help="BASELINE.json config (3 = the headline workload; 4, 5 = the larger-tile / 4M-vocab ones)")
    ap.add_argument("--sync-period", type=int, default=SYNC_P, help="words per GPU between model averagings")
    ap.add_argument("--sync-hot-rows", type=int, default=0,
                    help="C14 hot prefix averaged every interval (0 = all rows: C13, the default)")
    ap.add_argument("--sync-cold-every", type=int, default=1,
                    help="C14 cold rows averaged every this many intervals (1 = every interval: C13)")
    ap.add_argument("--sync-overlap", type=int, default=0, help="C15 overlapped averaging (1 = on)")
    ap.add_argument("--sync-device", type=int, default=0,
                    help="C17: each average as one kernel over NCCL symmetric memory (NVLS multimem when "
                         "available, else NVLink loads/stores) instead of ncclAllReduce (1 = on)")
    ap.add_argument("--scatter-wait", type=int, default=-1,
                    help="1: each target waits for its reductions to complete (R11); 0: only until read "
                         "(Hogwild staleness inside a chunk); -1: library default")
    ap.add_argument("--algorithm", choices=["hogbatch", "alg1"], default="hogbatch",
                    help="alg1: the paper's level-1 baseline (PAPER.md:37-63), for the HogBatch/Alg.1 ratio")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
