"""Gather-engine comparison on this GPU (SURVEY.md §8(a) "Gather engines"):
tools/libw2v_peaks.so peaks_gather_engines — random 1200-B rows (D = 300) of an L2-resident
working set gathered into shared memory by (0) one cp.async.bulk per row, (1) LSU ld.global.cg.v4
+ st.shared, (2) cp.async.cg 16-B (LDGSTS), (3) TMA tile::gather4; gather only, then gather +
bulk reduce-add back (the step kernel's per-target pattern). Prints one JSON line.

usage: python tools/engines.py [R] [units_per_sm]
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    units = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libw2v_peaks.so"))
    names = ["bulk cp.async.bulk per row", "LSU ld.global.cg.v4", "LDGSTS cp.async.cg", "TMA tile::gather4"]
    res = {"R_rows_per_batch": R, "units_per_sm": units, "row_bytes": 1200}
    out = (ctypes.c_double * 8)()
    bad = (ctypes.c_int * 4)()
    res["rc"] = lib.peaks_gather_engines(R, units, out, bad)
    res["engines"] = {names[e]: {"gather_GBps": out[e], "gather_plus_reduce_GBps": out[4 + e],
                                 "data_check_mismatches": bad[e]} for e in range(4)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
