import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
lib = ctypes.CDLL(os.path.join(os.getcwd(), "tools/libw2v_peaks.so"))
out = {}
for ns in (0, 3, 6, 8, 11):
    g = ctypes.c_double(0)
    rc = lib.peaks_l2_rowpath_store(1200, 11, 11, ns, ctypes.byref(g))
    out[ns] = round(g.value, 1) if rc == 0 else f"rc {rc}"
print(json.dumps({"rowpath_gbs_by_n_store_of_11": out}))
