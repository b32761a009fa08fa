"""World-size-2 gloo tests of the data-parallel protocol on CPU (C13, §7).

The B200 path averages replicas with NCCL; here two processes run the oracle's replica
protocol over torch.distributed/gloo. Checked: the union of the ranks' batch streams is
bit-identical to the 1-replica run (RNG keys are global positions), replicas are bit-identical
after every sync, W=1 equals the plain run, and the library's shard planner (pure host code,
no GPU) agrees with the protocol on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import inputs
import oracle
from oracle import dist as odist

V, D, WINDOW, K, T_SUB, L, SEED, P = 300, 8, 3, 4, 1e-3, 50, 77, 2_000
N_TOK = 23_456


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, hot_rows=0, cold_every=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = inputs.Corpus("iid", V, 1.0, SEED).tokens(0, N_TOK, threads=1)
    # global histogram = allreduce(sum) of the shard histograms (the B200 path does this in NCCL)
    lo, hi = odist.shard_chunks(N_TOK, L, world, rank)
    start, end = lo * L, min(hi * L, N_TOK)
    c_local = torch.from_numpy(oracle.counts(ids[start:end], V))
    dist.all_reduce(c_local, op=dist.ReduceOp.SUM)
    nsync = [0]
    max_disc = [0.0]

    def average(M_in, M_out):
        for M in (M_in, M_out):
            t = torch.from_numpy(M)   # a row-slice view when C14 averages only the hot prefix
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= world
            g = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(g, t)
            max_disc[0] = max(max_disc[0], max(float((x - t).abs().max()) for x in g))
        nsync[0] += 1

    M_in, M_out, st, dbg = odist.train_replica(ids, V, D, WINDOW, K, 0.025, T_SUB, SEED, L, world, rank, P,
                                                average, counts_global=c_local.numpy(), debug=(start, end - start),
                                                hot_rows=hot_rows, cold_every=cold_every)
    plan = None
    try:
        from paper_1611_06172_b200 import binding
        plan = binding.dist_plan(N_TOK, L, world, rank, P)
    except (ImportError, OSError):
        pass
    np.savez(os.path.join(outdir, f"r{rank}.npz"), M_in=M_in, M_out=M_out, keep=dbg.keep, b=dbg.b, N=dbg.N,
             ctx=dbg.ctx, neg=dbg.neg, nsync=nsync[0], disc=max_disc[0], words=st["words"],
             plan=np.asarray(plan if plan is not None else [], np.int64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("hot_rows,cold_every", [(0, 1), (60, 3)])
def test_two_replicas_gloo(tmp_path, hot_rows, cold_every):
    """C13 (full average after every interval) and C14 (hot prefix every interval, cold rows
    every 3rd and the last): union of streams == 1 replica, replicas identical at the end."""
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path), hot_rows, cold_every), nprocs=world,
                       join=True, start_method="spawn")
    r = [np.load(os.path.join(tmp_path, f"r{k}.npz")) for k in range(world)]
    ids = inputs.Corpus("iid", V, 1.0, SEED).tokens(0, N_TOK, threads=1)
    _, _, st1, dbg1 = oracle.train(ids, V, D, WINDOW, K, 0.025, T_SUB, SEED, L, debug=(0, N_TOK))
    # union of shard batch streams == single-replica stream, bit for bit
    for f in ("keep", "b", "N", "ctx", "neg"):
        assert np.array_equal(np.concatenate([x[f] for x in r]), getattr(dbg1, f)), f
    assert sum(int(x["words"]) for x in r) == st1["words"] == N_TOK
    # replicas identical after the final sync, and sync counts identical
    assert np.array_equal(r[0]["M_in"], r[1]["M_in"]) and np.array_equal(r[0]["M_out"], r[1]["M_out"])
    J = len(odist.sync_intervals(N_TOK, L, world, 0, P))
    assert int(r[0]["nsync"]) == int(r[1]["nsync"]) == J
    full = sum(odist.synced_rows(k, J, V, hot_rows, cold_every) == [(0, V)] for k in range(J))
    assert full == (J if hot_rows == 0 else len([k for k in range(J) if (k + 1) % cold_every == 0 or k == J - 1]))
    assert float(r[0]["disc"]) == 0.0
    # the library's host planner (if built) matches the protocol on both ranks
    for k in range(world):
        plan = r[k]["plan"]
        if plan.size:
            iv = odist.sync_intervals(N_TOK, L, world, k, P)
            assert [tuple(x) for x in plan.reshape(-1, 2)] == iv


def test_w1_equals_plain():
    ids = inputs.Corpus("iid", V, 1.0, SEED).tokens(0, N_TOK, threads=1)
    a_in, a_out, st_a, _ = oracle.train(ids, V, D, WINDOW, K, 0.025, T_SUB, SEED, L)
    calls = []
    b_in, b_out, st_b, _ = odist.train_replica(ids, V, D, WINDOW, K, 0.025, T_SUB, SEED, L, 1, 0, P,
                                               lambda a, b: calls.append(1))
    assert not calls
    assert np.array_equal(a_in, b_in) and np.array_equal(a_out, b_out)
    assert st_a == st_b


def test_shard_plan_partitions():
    for n, L_, W in [(1000, 20, 3), (23_456, 50, 8), (10, 20, 4), (1 << 20, 20, 8)]:
        S = (n + L_ - 1) // L_
        got = [odist.shard_chunks(n, L_, W, r) for r in range(W)]
        assert got[0][0] == 0 and got[-1][1] == S
        assert all(got[i][1] == got[i + 1][0] for i in range(W - 1))
        J = {len(odist.sync_intervals(n, L_, W, r, 4096)) for r in range(W)}
        assert len(J) == 1


def _loss_worker(rank, world, port, outdir, hot_rows, cold_every, overlap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Vg, n = 2000, 480_000
    ids = inputs.Corpus("iid", Vg, 1.0, 5).tokens(0, n, threads=1)
    c = oracle.counts(ids, Vg)

    def average(M_in, M_out):
        for M in (M_in, M_out):
            t = torch.from_numpy(M)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            t /= world

    M_in, M_out, st, _ = odist.train_replica(ids, Vg, 32, 5, 5, 0.025, 1e-3, 11, 20, world, rank, 1 << 11,
                                             average, counts_global=c, hot_rows=hot_rows, cold_every=cold_every,
                                             overlap=overlap)
    if rank == 0:
        held = inputs.Corpus("iid", Vg, 1.0, 5).tokens(n, 60_000, threads=1)
        _, _, hs, _ = oracle.train(held, Vg, 32, 5, 5, 0.0, 1e-3, 12, 20, model=(M_in, M_out))
        np.save(os.path.join(outdir, f"loss_{hot_rows}_{cold_every}_{int(overlap)}.npy"), hs["loss_sum"] / hs["loss_pairs"])
    # the replicas end identical (every protocol ends an epoch with a plain mean)
    g = [torch.empty_like(torch.from_numpy(M_in)) for _ in range(world)]
    dist.all_gather(g, torch.from_numpy(M_in))
    assert all(torch.equal(x, g[0]) for x in g)
    dist.barrier()
    dist.destroy_process_group()


def test_hot_cold_averaging_loss_gate(tmp_path):
    """C14/C15 change the sync semantics (SURVEY.md §8(f) NEXT-2 "gate it on loss"): 4 oracle
    replicas (58 sync intervals each) with the hot 10% of rows averaged every interval and the rest
    every 4th, with the bench's N > 1 default (hot 5%, the rest every 32nd and at the end), and
    with C15's one-interval-late (overlapped) averaging, reach a held-out SGNS loss within 1% of
    C13's full averaging after every interval; replicas end identical."""
    world = 4
    out = {}
    for hot, every, ovl in ((0, 1, False), (200, 4, False), (100, 32, False), (100, 32, True), (0, 1, True)):
        mp.start_processes(_loss_worker, args=(world, _free_port(), str(tmp_path), hot, every, ovl), nprocs=world,
                           join=True, start_method="spawn")
        out[(hot, every, ovl)] = float(np.load(os.path.join(tmp_path, f"loss_{hot}_{every}_{int(ovl)}.npy")))
    print("held-out loss/pair, 4 replicas: " + ", ".join(f"H={h} C={c} overlap={o}: {v:.6f}"
                                                         for (h, c, o), v in out.items()))
    for key in out:
        assert abs(out[key] / out[(0, 1, False)] - 1) < 0.01, key
