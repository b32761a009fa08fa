# tools/gpu_matrix.sh — ring kernel residency experiment (round 2)
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ring" > gpurun_out/pt_n.log 2>&1; echo "rc $?" >> gpurun_out/pt_n.log
timeout 600 python bench.py --kernel 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_n_r11.log 2>&1
W2V_LIBRARY=paper_1611_06172_b200/libw2v_ring8.so timeout 600 python bench.py --kernel 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_n_r8.log 2>&1
W2V_LIBRARY=paper_1611_06172_b200/libw2v_ring10.so timeout 600 python bench.py --kernel 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_n_r10.log 2>&1
