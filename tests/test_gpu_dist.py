"""Multi-GPU data-parallel parity (DESIGN.md §2 C13-C15): W processes, one
GPU each, train their C13 shards through the C-ABI in deterministic mode with the library's NCCL
model averaging; every rank's replica is compared with the oracle's replica protocol
(oracle/dist.py, fp64, run by the same rank over a gloo group), and the replicas must be
bit-identical to each other after the final average.

W = 2 needs two visible GPUs and skips cleanly otherwise; W = 1 runs the same worker with a
1-rank NCCL communicator (the plumbing check that runs on every one-GPU box).
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from test_gpu_parity import rel_l2, row_rel_max

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2])
@pytest.mark.parametrize("hot,cold_every,overlap,sync_device", [(0, 1, 0, 0), (150, 3, 0, 0), (0, 1, 1, 0),
                                                               (0, 1, 0, 1), (150, 3, 0, 1), (0, 1, 1, 1)])
def test_replicas_match_oracle_protocol(tmp_path, world, hot, cold_every, overlap, sync_device):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (visible: {torch.cuda.device_count()})")
    import __graft_entry__
    __graft_entry__.build_library()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(HERE, "dist_gpu_worker.py"), "--out", str(tmp_path), "--hot", str(hot),
           "--cold-every", str(cold_every), "--overlap", str(overlap), "--sync-device", str(sync_device)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"gpu_r{k}.npz")) for k in range(world)]
    for k, x in enumerate(res):
        for f in ("words", "targets", "row_touches"):
            assert int(x[f]) == int(x["o_" + f]), (k, f)
        J = int(x["J"])
        assert int(x["syncs"]) + int(x["syncs_hot"]) == J  # one average per interval (C13/C14/C15)
        assert int(x["sync_path"]) in ((2, 3) if sync_device else (1,))  # C17 kernel (LSA or NVLS) / NCCL
        for name, g, o in (("M_in", x["M_in"], x["o_in"]), ("M_out", x["M_out"], x["o_out"])):
            e, rr = rel_l2(g, o), row_rel_max(g, o)
            print(f"W={world} H={hot} C={cold_every} overlap={overlap} rank {k} {name}: rel L2 {e:.3e}, "
                  f"per-row max {rr:.3e}, J={J}")
            assert e <= 1e-5
            assert rr <= 1e-4
    # every protocol ends the epoch with a plain mean: the replicas are bit-identical
    for x in res[1:]:
        assert np.array_equal(x["M_in"], res[0]["M_in"]) and np.array_equal(x["M_out"], res[0]["M_out"])
