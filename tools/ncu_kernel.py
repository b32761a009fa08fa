"""Print selected metrics of every kernel in an ncu report (details + raw pages).

usage: python tools/ncu_kernel.py REPORT.ncu-rep [substring-of-kernel-name] [--all-lts]
"""
import csv
import subprocess
import sys

DET = ['Duration', 'DRAM Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput', 'Issue Slots Busy',
       'L2 Hit Rate', 'Registers Per Thread', 'Achieved Active Warps Per SM', 'Eligible Warps Per Scheduler',
       'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Dynamic Shared Memory Per Block']
RAW = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors_srcunit_tex_op_red.sum',
       'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed',
       'lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed',
       'lts__t_sectors.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors.max.pct_of_peak_sustained_elapsed',
       'lts__t_sectors_srcunit_ltcfabric.sum', 'l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed',
       'l1tex__m_l1tex2xbar_write_bytes.sum.pct_of_peak_sustained_elapsed',
       'dram__cycles_active.max.pct_of_peak_sustained_elapsed', 'lts__t_sector_op_read_hit_rate.pct',
       'lts__t_sector_op_write_hit_rate.pct', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
       'gpu__time_duration.sum']


def main(rep, sub=""):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(det.splitlines())
    h = next(r)
    out = {}
    for row in r:
        d = dict(zip(h, row))
        if sub in d["Kernel Name"] and d["Metric Name"] in DET:
            out.setdefault((d["ID"], d["Kernel Name"][:60]), {})[d["Metric Name"]] = d["Metric Value"] + " " + d["Metric Unit"]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hh, uu = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(hh, row))
        key = (d["ID"], d["Kernel Name"][:60])
        if key in out:
            for k in RAW:
                if k in d:
                    out[key][k] = d[k] + " " + uu[hh.index(k)]
    for k, v in out.items():
        print(k)
        for m, x in v.items():
            print(f"   {m:75s} {x}")


if __name__ == "__main__":
    main(*sys.argv[1:])
