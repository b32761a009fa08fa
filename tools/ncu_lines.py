"""Summarise an ncu report per CUDA source line: instructions executed and warp-stall samples."""
import csv
import os
import subprocess
import sys

# kernel filter for multi-kernel reports (the step kernel by default)
KFILT = os.environ.get("W2V_NCU_KERNEL", "regex:hogbatch_step")


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "-k", KFILT, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    hdr = None
    lines = []
    cur = "?"
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1]
            continue
        if len(r) > 5 and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] not in ("",):
            d = dict(zip(hdr, r))
            try:
                ln = int(d["Line No"])
                src = ""
                try:
                    src = open(cur).read().splitlines()[ln - 1]
                except (OSError, IndexError):
                    pass
                lines.append((f"{os.path.basename(cur)}:{ln}", src[:90], int(d["Warp Stall Sampling (All Samples)"] or 0),
                              int(d["Instructions Executed"] or 0),
                              {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k
                               and v.isdigit() and int(v) > 0}))
            except (ValueError, KeyError):
                pass
    tot_s = sum(x[2] for x in lines) or 1
    tot_i = sum(x[3] for x in lines) or 1
    print(f"total samples {tot_s}, instructions {tot_i}")
    for ln, src, s, i, st in sorted(lines, key=lambda x: -x[2])[:top]:
        reasons = ", ".join(f"{k[6:]}={v * 100 // max(s, 1)}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{ln:24s} {100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% inst | {src.strip()[:60]:60s} | {reasons}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
