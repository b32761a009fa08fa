"""Executed-instruction mix by SASS opcode from an ncu report's source page."""
import collections
import csv
import os
import subprocess
import sys

# kernel filter for multi-kernel reports (the step kernel by default)
KFILT = os.environ.get("W2V_NCU_KERNEL", "regex:hogbatch_step")

out = subprocess.run(["ncu", "-i", sys.argv[1], "-k", KFILT, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
cnt = collections.Counter()
for r in rows:
    if len(r) > 5 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        src = d["Source"].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        try:
            cnt[op] += int(d["Instructions Executed"] or 0)
        except ValueError:
            pass
tot = sum(cnt.values())
print("total", tot)
for op, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:12s} {100 * c / tot:5.1f}%")
