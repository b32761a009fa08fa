"""Time one C17 model average (sync_dev.cu) against the NCCL all-reduce path on the cfg3 model
(V = 1M, D = 300: 2.4 GB) on a 1-rank communicator — the only communicator a one-GPU box can
build. At W = 1 both are the identity: NCCL still copies the buffer in place, the C17 kernel streams the
model through the LSA path (load + store of every float, 2 x 2.4 GB): this measures its HBM
efficiency and launch/barrier overhead, not NVLink. Prints one JSON line.

    python tools/sync_dev_bw.py [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--V", type=int, default=1_000_000)
    ap.add_argument("--D", type=int, default=300)
    a = ap.parse_args()
    from paper_1611_06172_b200 import binding as w2v
    out = {}
    for dev in (0, 1):
        w2v.init(a.V, a.D, 5, 5, 0.025, 1e-4, 1)
        w2v.set_option("sync_device", dev)
        w2v.dist_init(0, 1, w2v.dist_unique_id())
        s = torch.cuda.current_stream()
        w2v.set_stream(s.cuda_stream)
        w2v.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(a.reps):
            w2v.sync()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        st = w2v.get_stats()
        Ds = (a.D + 31) // 32 * 32
        model_bytes = a.V * 2 * Ds * 4
        out["c17_kernel" if dev else "nccl_allreduce"] = {
            "ms": ms, "sync_path": st["sync_path"], "model_bytes": model_bytes,
            "GBps_read_plus_write": 2 * model_bytes / ms / 1e6 if dev else None,
            "floats_owned": st["sync_floats_owned"]}
        w2v.finalize()
    print(json.dumps({"tool": "sync_dev_bw", "world": 1, **out}))


if __name__ == "__main__":
    main()
