"""Key metrics of an ncu report (details + raw pages) as JSON-able dict and a printed table."""
import csv
import json
import os
import subprocess
import sys

# kernel filter for multi-kernel reports (the step kernel by default)
KFILT = os.environ.get("W2V_NCU_KERNEL", "regex:hogbatch_step")

DETAILS = ['Duration', 'DRAM Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput', 'Executed Ipc Active',
           'Issue Slots Busy', 'L2 Hit Rate', 'Registers Per Thread', 'Achieved Active Warps Per SM',
           'Theoretical Active Warps per SM', 'Executed Instructions', 'No Eligible', 'Eligible Warps Per Scheduler',
           'Warp Cycles Per Issued Instruction', 'L1/TEX Hit Rate', 'Block Limit Registers', 'Block Limit Shared Mem']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'gpu__time_duration.sum',
       'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
       'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
       'l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum', 'lts__t_sectors_op_red.sum',
       'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
       'lts__t_sectors_srcunit_tex_op_red.sum', 'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed',
       'lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed',
       'lts__t_sectors.max.pct_of_peak_sustained_elapsed',
       'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
       'l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed',
       'dram__cycles_active.max.pct_of_peak_sustained_elapsed', 'lts__t_sectors_srcunit_ltcfabric.sum']


def summary(rep):
    out = {}
    det = subprocess.run(["ncu", "-i", rep, "-k", KFILT, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(det.splitlines())
    hdr = next(r)
    for row in r:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") in DETAILS:
            out[d["Metric Name"]] = (d["Metric Value"], d["Metric Unit"])
    raw = subprocess.run(["ncu", "-i", rep, "-k", KFILT, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    for h, u, v in zip(rows[0], rows[1], rows[-1]):
        if h in RAW:
            out[h] = (v, u)
    return out


if __name__ == "__main__":
    s = summary(sys.argv[1])
    for k, (v, u) in s.items():
        print(f"{k:62s} {u:14s} {v}")
    if len(sys.argv) > 2:
        json.dump({k: {"value": v, "unit": u} for k, (v, u) in s.items()}, open(sys.argv[2], "w"), indent=1)
