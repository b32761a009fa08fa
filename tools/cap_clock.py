import ctypes, os, subprocess, threading, time, json
lib = ctypes.CDLL(os.path.join(os.getcwd(), "tools/libw2v_peaks.so"))
def sample(out, stop):
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        out.append(r); time.sleep(0.2)
res = {}
for nb in (2000, 40000):
    os.environ["W2V_CAP_BATCHES"] = str(nb)
    g = ctypes.c_double(0); samples = []; stop = threading.Event()
    th = threading.Thread(target=sample, args=(samples, stop)); th.start()
    t0 = time.time(); rc = lib.peaks_l2_rowpath(1200, 11, 11, ctypes.byref(g)); dt = time.time() - t0
    stop.set(); th.join()
    res[nb] = {"gbs": round(g.value, 1), "wall_s": round(dt, 2), "clock_power_samples": samples[-5:]}
print(json.dumps(res))
