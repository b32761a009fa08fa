"""Row-path cap (tools/peaks.cu peaks_l2_rowpath_store) vs row size: is a partial last sector
(1200-B rows) slower per row than whole 128-B lines (1280 B)? Prints rows/s and GB/s."""
import ctypes, json, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libw2v_peaks.so"))
out = {}
for rb in (1152, 1200, 1216, 1280):
    for ns in (0, 11):
        g = ctypes.c_double(0)
        rc = lib.peaks_l2_rowpath_store(rb, 11, 11, ns, ctypes.byref(g))
        out[f"{rb}B_{'store' if ns else 'reduce'}"] = {"gbs": round(g.value, 1), "Grows_s": round(g.value / rb / 2, 3)} if rc == 0 else rc
print(json.dumps(out))
