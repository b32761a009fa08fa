"""The in-run roofline denominators bench.py measures (tools/peaks.cu), printed as one JSON line —
and the command profiles/r02_l2cap_ncu.* runs under ncu to record the L2 slice counters of the
cap pattern (lts__t_sectors.sum, lts__cycles_elapsed.avg, lts__d_atomic_input_cycles_active).

usage: python tools/caps.py [row_bytes] [rows_per_batch] [units_per_sm]
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rb = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    units = int(sys.argv[3]) if len(sys.argv) > 3 else 11
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libw2v_peaks.so"))
    d = ctypes.c_double(0.0)
    out = {"row_bytes": rb, "rows_per_batch": R}
    for w in sorted({units, 8, 12, 16}):
        if lib.peaks_l2_rowpath(rb, R, w, ctypes.byref(d)) == 0:
            out[f"l2_rowpath_gbs_units{w}"] = d.value
    for name, fn in (("ffma2_tflops", lib.peaks_ffma2), ("l2_read_gbs", lib.peaks_l2_read),
                     ("l2_red_gbs", lib.peaks_l2_red)):
        if fn(ctypes.byref(d)) == 0:
            out[name] = d.value
    print(json.dumps(out))


if __name__ == "__main__":
    main()
