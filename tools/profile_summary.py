"""Write the per-round profile summaries under profiles/ from gpurun_out/ artefacts.

usage: python tools/profile_summary.py r01 gpurun_out/launches_r01.csv gpurun_out/prof_r01.ncu-rep \
           gpurun_out/bench_default.log
Produces profiles/<tag>_launches.md (kernel shares of the bench command's launch list),
profiles/<tag>_hogbatch_step_ncu.md/.json (key metrics, stall lines, opcode mix) and updates
profiles/ncu_traffic.json (DRAM bytes per raw word of the captured launch, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}[d["Metric Unit"]]
            name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "")
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"]) * scale
    return agg


def main(tag, csv_path, rep, bench_log):
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    bench = json.loads([ln for ln in open(bench_log).read().splitlines() if ln.startswith("{")][-1])
    agg = launches(csv_path)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list of `python bench.py` (gpu__time_duration.sum, --clock-control none)\n\n")
        f.write("Cold-cache, serialised per-launch times: compare SHARES with the bench, not absolutes.\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {ms:.2f} | {100 * ms / tot:.2f}% |\n")
        f.write(f"\nBench (no profiler): kernel_share_of_step = {bench['roofline']['kernel_share_of_step']:.4f}, "
                f"value = {bench['value'] / 1e6:.1f} M words/s, L2 row-path fraction = {bench['roofline']['frac']:.3f}, "
                f"R_HBM = {bench['roofline_hbm']['frac']:.3f}.\n")
    s = ncu_summary.summary(rep)
    dram = float(s["dram__bytes_read.sum"][0]) + float(s["dram__bytes_write.sum"][0])
    unit = s["dram__bytes_read.sum"][1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    dram_bytes = dram * mult
    words = int(os.environ.get("W2V_PROFILED_WORDS", str(1 << 26)))
    # L2 slice (LTS) throughput of the capture: all LTS sectors / LTS cycles, chip-wide B/cycle —
    # against the LTS cap /opt/skills/guides/B300_MICROARCH.md measures (~6300 B/cycle full-chip)
    raw = subprocess.run(["ncu", "-i", rep, "-k", os.environ.get("W2V_NCU_KERNEL", "regex:hogbatch_step"), "--page",
                          "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rd = dict(zip(rr[0], rr[-1]))
    lts_bpc = float(rd["lts__t_sectors.sum"]) * 32 / float(rd["lts__cycles_elapsed.avg"])
    traffic = {"dram_bytes_per_launch": dram_bytes, "words_per_launch": words,
               "dram_bytes_per_word": dram_bytes / words, "source": os.path.basename(rep), "round": tag,
               "algorithmic_bytes_per_word": bench["roofline_hbm"]["row_bytes_per_word"],
               "config": int(os.environ.get("W2V_PROFILED_CONFIG", "3")), "kernel": "hogbatch_step (rows)",
               "kernel_id": 1, "lts_bytes_per_cycle": lts_bpc,
               "lts__t_sectors.sum": float(rd["lts__t_sectors.sum"]),
               "lts__cycles_elapsed.avg": float(rd["lts__cycles_elapsed.avg"])}
    cap = os.path.join(ROOT, "profiles", "r02_l2cap_ncu.json")
    if os.path.exists(cap):
        c = json.load(open(cap))
        best = max(x["lts_bytes_per_cycle"] for x in c["rowpath_cap_ncu"])
        traffic["lts_cap_bytes_per_cycle"] = best
        traffic["lts_frac_of_cap"] = lts_bpc / best
        traffic["lts_cap_source"] = ("measured: tools/peaks.cu peaks_l2_rowpath under ncu (bulk gather of 11 rows + "
                                     "bulk reduce, 1200-B rows, L2-resident; best residency), profiles/r02_l2cap_ncu.json")
    json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
    json.dump({k: {"value": v, "unit": u} for k, (v, u) in s.items()},
              open(os.path.join(ROOT, "profiles", f"{tag}_hogbatch_step_ncu.json"), "w"), indent=1)
    lines = io.StringIO()
    with redirect_stdout(lines):
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"], check=True)
    ops = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_opcodes.py"), rep, "20"],
                         capture_output=True, text=True).stdout
    lines_out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "25"],
                               capture_output=True, text=True).stdout
    with open(os.path.join(ROOT, "profiles", f"{tag}_hogbatch_step_ncu.md"), "w") as f:
        f.write(f"# {tag}: `ncu --set full` of one hogbatch_step launch ({words} raw words of cfg3)\n\n")
        cmd = os.environ.get("W2V_PROFILED_CMD", "ncu --set full --clock-control none --import-source on "
                             "-k regex:hogbatch_step -s 5 -c 1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline")
        f.write(f"Command: `{cmd}` (after the same command exited 0).\n\n")
        f.write("| metric | unit | value |\n|---|---|---|\n")
        for k, (v, u) in s.items():
            f.write(f"| {k} | {u} | {v} |\n")
        f.write(f"\nDRAM traffic per launch = {dram_bytes / 1e9:.1f} GB = {dram_bytes / words:.0f} B per raw word "
                f"(algorithmic row bytes {bench['roofline_hbm']['row_bytes_per_word']:.0f} B/word: L2 serves "
                f"{100 * (1 - dram_bytes / words / bench['roofline_hbm']['row_bytes_per_word']):.0f}% of the row traffic).\n")
        f.write(f"\nL2 slices: lts__t_sectors.sum = {float(rd['lts__t_sectors.sum']):.4g}, lts__cycles_elapsed.avg = "
                f"{float(rd['lts__cycles_elapsed.avg']):.4g} -> {lts_bpc:.0f} B per L2 cycle chip-wide"
                + (f" = {traffic['lts_frac_of_cap']:.3f} of the cap pattern's {traffic['lts_cap_bytes_per_cycle']:.0f} "
                   f"(profiles/r02_l2cap_ncu.json)" if "lts_frac_of_cap" in traffic else "") + ".\n")
        f.write("\n## Warp-stall samples by source line (top 25)\n\n```\n" + lines_out + "```\n")
        f.write("\n## Executed instruction mix (SASS opcodes)\n\n```\n" + ops + "```\n")
    print(open(os.path.join(ROOT, "profiles", f"{tag}_launches.md")).read())
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:5])
