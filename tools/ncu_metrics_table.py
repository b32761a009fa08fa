"""Per-launch table of an `ncu --metrics ... --csv` log (the lines after the program's own
output): one row per kernel launch with the L2 slice counters used by DESIGN.md §8 — sectors,
sectors per L2 cycle (chip), reduction sectors, fabric (cross-die) sectors, atomic-unit activity.

usage: python tools/ncu_metrics_table.py gpurun_out/engines_ncu.csv [md]
"""
import csv
import io
import sys


def launches(path):
    txt = open(path).read()
    i = txt.find('"ID","Process ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    out = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void <unnamed>::", ""))
        out.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return out


def main():
    L = launches(sys.argv[1])
    md = len(sys.argv) > 2
    hd = ["launch", "kernel", "time ms", "L2 sectors G", "B/L2-cycle", "red sectors G", "fabric sectors G",
          "atomic unit %", "DRAM GB"]
    print("| " + " | ".join(hd) + " |" if md else "\t".join(hd))
    if md:
        print("|" + "---|" * len(hd))
    for (i, name), m in sorted(L.items()):
        t = m.get("gpu__time_duration.sum", 0) / 1e6
        sec = m.get("lts__t_sectors.sum", 0)
        cyc = m.get("lts__cycles_elapsed.avg", 1)
        row = [str(i), name, f"{t:.3f}", f"{sec / 1e9:.3f}", f"{sec * 32 / cyc:.0f}",
               f"{m.get('lts__t_sectors_op_red.sum', 0) / 1e9:.3f}",
               f"{m.get('lts__t_sectors_srcunit_ltcfabric.sum', 0) / 1e9:.3f}",
               f"{m.get('lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f}",
               f"{(m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e9:.3f}"]
        print("| " + " | ".join(row) + " |" if md else "\t".join(row))


if __name__ == "__main__":
    main()
