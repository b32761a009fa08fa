"""One rank of the multi-GPU replica test (tests/test_gpu_dist.py), launched by torchrun.

Each rank trains its C13 shard through the C-ABI on its own GPU in deterministic mode with the
library's NCCL model averaging (C13 full average, C14 hot/cold, or C15 overlapped), then runs
the ORACLE's replica protocol (oracle/dist.py train_replica, fp64, averaging over a gloo group
on the host) for the same rank, and saves both models plus the comparison. PAPER.md:154-157
(data parallelism), :186 (model synchronisation frequency); DESIGN.md §2 C13-C15.

TEST INFRASTRUCTURE ONLY (it imports oracle/).
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import inputs  # noqa: E402
import oracle  # noqa: E402
from oracle import dist as odist  # noqa: E402

# small shapes: the fp64 oracle replica must finish in seconds; several tiles and a ragged shard
V, D, WINDOW, K, T_SUB, L, SEED = 2000, 64, 3, 4, 1e-3, 50, 91
ALPHA = 0.025


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--n", type=int, default=60_123)
    ap.add_argument("--period", type=int, default=5_000)
    ap.add_argument("--hot", type=int, default=0)
    ap.add_argument("--cold-every", type=int, default=1)
    ap.add_argument("--overlap", type=int, default=0)
    ap.add_argument("--sync-device", type=int, default=0)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")   # host group: the NCCL id broadcast and the oracle's averages

    from paper_1611_06172_b200 import binding as w2v
    ids = inputs.Corpus("iid", V, 1.0, SEED).tokens(0, a.n, threads=1)
    start, end = w2v.dist_shard(a.n, L, world, rank)
    w2v.init(V, D, WINDOW, K, ALPHA, T_SUB, SEED)
    w2v.set_option("mode", 1)                      # deterministic (conflict-serialised) per replica
    w2v.set_option("sentence_len", L)
    w2v.set_option("sync_period_words", a.period)
    w2v.set_option("sync_hot_rows", a.hot)
    w2v.set_option("sync_cold_every", a.cold_every)
    w2v.set_option("sync_overlap", a.overlap)
    w2v.set_option("sync_device", a.sync_device)   # C17: the average as one kernel (sync_dev.cu)
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(w2v.dist_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    w2v.dist_init(rank, world, bytes(uid.numpy().tolist()))   # a real NCCL communicator (also at W=1)
    shard = torch.from_numpy(np.ascontiguousarray(ids[start:end])).cuda()
    w2v.train(shard, end - start, 1)
    g_in = np.empty((V, D), np.float32)
    g_out = np.empty((V, D), np.float32)
    w2v.get_embeddings(0, g_in)
    w2v.get_embeddings(1, g_out)
    st = w2v.get_stats()
    w2v.finalize()

    # the oracle's replica r of W: global counts, same shard and intervals, fp64 averages
    c = oracle.counts(ids, V)

    def average(M_in, M_out):
        for M in (M_in, M_out):
            t = torch.from_numpy(M)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= world

    o_in, o_out, o_st, _ = odist.train_replica(ids, V, D, WINDOW, K, ALPHA, T_SUB, SEED, L, world, rank, a.period,
                                               average, counts_global=c, hot_rows=a.hot, cold_every=a.cold_every,
                                               overlap=bool(a.overlap))
    J = len(odist.sync_intervals(a.n, L, world, rank, a.period))
    np.savez(os.path.join(a.out, f"gpu_r{rank}.npz"), M_in=g_in, M_out=g_out, o_in=o_in, o_out=o_out,
             words=st["words"], targets=st["targets"], row_touches=st["row_touches"], syncs=st["syncs"],
             syncs_hot=st["syncs_hot"], o_words=o_st["words"], o_targets=o_st["targets"],
             o_row_touches=o_st["row_touches"], J=J, sync_path=st["sync_path"])
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
