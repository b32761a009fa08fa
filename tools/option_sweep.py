"""Sweep library options on one workload (default cfg3, Hogwild, full size): words/s of the timed
w2v_train calls (CUDA events on the library's stream) per option setting, one JSON line.

    python tools/option_sweep.py --config 3 --steps 2 l2_hot_rows=0,13107,26214,52428,104857,1000000
    python tools/option_sweep.py l2_hint=0,1,3
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("sweep", nargs="+", help="key=v1,v2,...")
    a = ap.parse_args()
    from paper_1611_06172_b200 import binding as w2v
    cfg = inputs.CONFIGS[a.config]
    dev = torch.empty(cfg.n, dtype=torch.int32, device="cuda")
    cfg.corpus().tokens_cuda(0, cfg.n, dev)
    torch.cuda.synchronize()
    out = {}
    for spec in a.sweep:
        key, vals = spec.split("=")
        for v in vals.split(","):
            w2v.init(cfg.V, cfg.D, cfg.window, cfg.K, cfg.alpha, cfg.t, cfg.seed)
            w2v.set_option("sentence_len", cfg.L)
            w2v.set_option(key, int(v))
            s = torch.cuda.current_stream()
            w2v.set_stream(s.cuda_stream)
            w2v.train(dev, cfg.n, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(a.steps):
                w2v.train(dev, cfg.n, 1)
            e1.record(s)
            torch.cuda.synchronize()
            out[f"{key}={v}"] = round(cfg.n * a.steps / (e0.elapsed_time(e1) / 1e3) / 1e6, 2)
            w2v.finalize()
    print(json.dumps({"tool": "option_sweep", "config": a.config, "Mwords_per_s": out}))


if __name__ == "__main__":
    main()
