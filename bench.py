#!/usr/bin/env python
"""Benchmark: words/sec of the HogBatch SGNS step on BASELINE.json cfg3 (V=1M, D=300, 800M
planted Zipf(1.07) tokens, window=5, K=5, t=1e-4), 1..8 B200s, plus its gather/scatter HBM
roofline fraction.

A step = one `w2v_train(corpus, n, 1)` call = every SURVEY.md §8(a) row over the whole corpus
(setup a0, subsampling/window a1, sampler a2, fused step a3-a7, L2 window a8, and with N>1 the
model averaging a9 every 2^20 words per GPU). `value` is device-timed (CUDA events on the
library's stream, max over ranks) with the corpus resident in HBM; `e2e` is the same call with a
pinned HOST corpus (H2D inside the timed region). `--impl reference` times the CPU oracle.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
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
REF_SAMPLE = 1 << 17      # raw words per reference step (bounded CPU sample of cfg3)
BASE_SAMPLE = 1 << 19     # raw words for the cpu_baseline leg


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

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
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _oracle_setup(cfg, sample):
    import oracle
    ids = cfg.corpus().tokens(0, sample)
    c = oracle.counts(ids, cfg.V)
    thr, P = oracle.thresholds(c, sample, cfg.t), oracle.sampler(c)
    prm = oracle.make_params(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed, cfg.L, 1, sample)
    return ids, thr, P, prm


def _oracle_model(cfg):
    import oracle
    mi, mo = oracle.init(cfg.V, cfg.D, cfg.seed)
    M_in, M_out = mi.astype(np.float64), mo.astype(np.float64)
    return M_in, M_out


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:
        return max(1, os.cpu_count() or 1)


def cpu_baseline(cfg, sample):
    """The oracle as it stands on the box's host cores: its Hogwild threaded mode over all cores
    (the paper's CPU setting) on `threads` x `sample` raw words, plus
    the sequential fp64 O-HB on `sample` words as `value_1core`; setup excluded."""
    import oracle
    T = host_threads()
    ids, thr, P, prm = _oracle_setup(cfg, sample * T)
    n = sample * T
    prm = oracle.make_params(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed, cfg.L, 1, n)
    M_in, M_out = _oracle_model(cfg)
    nch = (n + cfg.L - 1) // cfg.L
    t0 = time.perf_counter()
    oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), T)
    dt_t = time.perf_counter() - t0
    del M_in, M_out
    M_in, M_out = _oracle_model(cfg)
    nch1 = (sample + cfg.L - 1) // cfg.L
    t0 = time.perf_counter()
    oracle.train_range(prm, thr, P, ids, 0, 0, n, 0, 0, nch1, M_in, M_out, oracle.OrcStats())
    dt_1 = time.perf_counter() - t0
    return {"value": n / dt_t, "unit": "words/s", "cores": T, "kind": "oracle",
            "sample": f"first {n} raw words of cfg{cfg.idx} (V={cfg.V}, D={cfg.D}), fp64 O-HB in the oracle's "
                      f"Hogwild threaded mode on {T} host threads, setup excluded",
            "seconds": dt_t, "value_1core": sample / dt_1,
            "sample_1core": f"first {sample} raw words, sequential fp64 O-HB, 1 thread ({dt_1:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = inputs.CONFIGS[CFG]
    import oracle
    T = host_threads()
    n = REF_SAMPLE * T
    ids, thr, P, prm = _oracle_setup(cfg, n)
    M_in, M_out = _oracle_model(cfg)
    nch = (n + cfg.L - 1) // cfg.L
    for _ in range(args.warmup):
        oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), T)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.train_range_hogwild(prm, thr, P, ids, 0, 0, n, 0, 0, nch, M_in, M_out, oracle.OrcStats(), T)
    dt = time.perf_counter() - t0
    v = n * args.steps / dt
    sample = (f"first {n} raw words of cfg3 per step, fp64 oracle (O-HB) in its Hogwild threaded mode on "
              f"{T} host threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "words/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 (bounded CPU sample)", "V": cfg.V, "D": cfg.D, "window": cfg.window,
                   "K": cfg.K, "t": cfg.t, "sample_words": n},
        "cpu_baseline": {"value": v, "unit": "words/s", "cores": T, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "words/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1611_06172_b200 import binding as w2v

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
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
    # C14 by default when N > 1: the hot 5% of the rows averaged every interval, the rest every
    # 32nd and at the end (C14 and §10: C13's full 2.4 GB average per 2^20 words would
    # dominate the step; the loss gate is tests/test_dist_gloo.py)
    hot = args.sync_hot_rows if args.sync_hot_rows >= 0 else (cfg.V // 20 if world > 1 else 0)
    cold = args.sync_cold_every if args.sync_cold_every > 0 else (32 if world > 1 else 1)
    w2v.set_option("sync_hot_rows", hot)      # 0 = C13 full averaging
    w2v.set_option("sync_cold_every", cold)
    ovl = int(args.sync_overlap > 0)   # C15 only on request (unmeasured at N > 1)
    w2v.set_option("sync_overlap", ovl)
    w2v.set_option("kernel", args.kernel)
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

    for _ in range(args.warmup):
        w2v.train(dev, n_local, 1)
    barrier()
    steps = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            w2v.train(dev, n_local, 1)
            steps.append(w2v.get_stats())
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    ms_step_kernel = sum(s["ms_step"] for s in steps) / len(steps)
    t = torch.tensor([ms, ms_step_kernel], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, kern_max = float(t[0]), float(t[1])
    value = n * args.steps / (ms_max / 1e3)

    # e2e: the same call with a pinned HOST corpus (H2D + stats D2H inside the timed region)
    e2e_steps = max(1, min(args.steps, 3))
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        w2v.train(host, n_local, 1)
    f1.record(stream)
    barrier()
    te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n * e2e_steps / (float(te[0]) / 1e3)
    last = steps[-1]

    # row-path roof: the same kernel and batch stream with a4-a6 skipped (zero deltas reduced,
    # model unchanged) — what the gathers + scatters alone sustain on this chip
    roof = None
    if args.algorithm == "hogbatch" and args.kernel in (0, 1):
        w2v.set_option("rowpath_only", 1)
        w2v.train(dev, n_local, 1)
        rs = w2v.get_stats()
        w2v.set_option("rowpath_only", 0)
        tr = torch.tensor([rs["ms_step"]], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        roof = n / (float(tr[0]) / 1e3)

    if rank == 0:
        peak, peak_src = peaks()
        achieved = last["bytes_row"] / (last["ms_step"] / 1e3) / 1e9   # GB/s, algorithmic bytes
        traffic = None   # DRAM bytes per launch (ncu --set full capture, profiles/), scaled to this launch size
        l2roof = None    # the binding resource per that capture: L2 slice (LTS) throughput
        prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(prof) and args.algorithm == "hogbatch" and args.kernel in (0, 1):
            tr = json.load(open(prof))
            if tr.get("config", 3) == args.config:  # the capture is of this workload and kernel
                traffic = tr.get("dram_bytes_per_word") * n_local / max(last["step_launches"], 1)
                if "lts_bytes_per_cycle" in tr:
                    l2roof = {"bound": "l2 (LTS slice throughput, all sectors incl. cross-die)",
                              "achieved": tr["lts_bytes_per_cycle"], "peak": tr["lts_cap_bytes_per_cycle"],
                              "unit": "B/cycle (chip)", "frac": tr["lts_bytes_per_cycle"] / tr["lts_cap_bytes_per_cycle"],
                              "source": f"ncu --set full capture {tr.get('source')} (profiles/); peak: "
                                        + tr.get("lts_cap_source", "")}
        out = {
            "metric": METRIC, "value": value, "unit": "words/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config],
                       "V": cfg.V, "D": cfg.D, "n_tokens": n, "full_size": n == cfg.n, "sync_period_words": args.sync_period if world > 1 else None,
                       "sync": (("C13 full average every interval" if hot == 0 else
                                 f"C14: rows [0,{hot}) averaged every interval, the rest every {cold}th and at the end")
                                + ("; C15: each average in flight during the next interval, applied one interval late"
                                   if ovl else "")) if world > 1 else None,
                       "parallelism": f"dp{world} corpus-sharded replicas" if world > 1 else "single GPU",
                       "l2": f"no flush: corpus ({n_local * 4 / 1e9:.1f} GB) and model ({cfg.V * cfg.D * 8 / 1e9:.2f} GB) exceed the 126 MB L2",
                       "units_per_sm": last["units_per_sm"], "mode": "hogwild", "kernel": {1: "rows", 2: "window", 3: "window-wg", 4: "alg1"}.get(last["kernel"]),
                       "algorithm": "hogbatch" if args.algorithm == "hogbatch" else "alg1 (PAPER.md:37-63, level-1 baseline)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "hogbatch_step" if args.algorithm == "hogbatch" else "alg1",
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": last["bytes_row"] / max(last["step_launches"], 1),
                         "row_bytes_per_word": last["bytes_row"] / n_local,
                         "kernel_ms_per_step": kern_max, "kernel_share_of_step": kern_max / (ms_max / args.steps)},
            "roofline_l2": l2roof,
            "rowpath_roof": None if roof is None else {
                "value": roof, "unit": "words/s", "frac": (n / (kern_max / 1e3)) / roof,
                "how": "same step kernel, launch configuration and batch stream with a4-a6 skipped (zero "
                       "deltas reduced): the gather/scatter path alone; frac = step-kernel words/s / roof"},
            "e2e": {"value": e2e_value, "unit": "words/s", "h2d_bytes_per_step": n_local * 4,
                    "d2h_bytes_per_step": 64},
            "gpu_launches": int(sum(s["launches"] for s in steps)),
            "clocks": clk.summary(),
            "stats": {"loss_per_pair": last["loss_sum"] / max(last["loss_pairs"], 1),
                      "ms_setup": last["ms_setup"], "ms_step": last["ms_step"], "ms_sync": last["ms_sync"],
                      "syncs": last["syncs"]},
        }
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
    ap.add_argument("--kernel", type=int, default=0,
                    help="0 auto, 1 per-target rows, 2 window-resident rows, 3 window-resident warp-specialised")
    ap.add_argument("--tokens", type=int, default=0, help="profiling only: train on a cfg3 prefix")
    ap.add_argument("--config", type=int, choices=[3, 4, 5], default=CFG,
                    help="BASELINE.json config (3 = the headline workload; 4, 5 = the larger-tile / 4M-vocab ones)")
    ap.add_argument("--sync-period", type=int, default=SYNC_P, help="words per GPU between model averagings")
    ap.add_argument("--sync-hot-rows", type=int, default=-1,
                    help="C14 hot prefix averaged every interval (0 = all rows, C13; -1 = V/20 when N > 1)")
    ap.add_argument("--sync-cold-every", type=int, default=0,
                    help="C14 cold rows averaged every this many intervals (0 = 32 when N > 1)")
    ap.add_argument("--sync-overlap", type=int, default=0, help="C15 overlapped averaging (1 = on)")
    ap.add_argument("--algorithm", choices=["hogbatch", "alg1"], default="hogbatch",
                    help="alg1: the paper's level-1 baseline (PAPER.md:37-63), for the HogBatch/Alg.1 ratio")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
