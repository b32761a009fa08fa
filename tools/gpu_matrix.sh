python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_v.log 2>&1
W2V_LIBRARY=paper_1611_06172_b200/libw2v_t6.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1_deterministic or (edge and (1 or 4)) or ring_det or headline" > gpurun_out/pt_v.log 2>&1; echo "rc $?" >> gpurun_out/pt_v.log
for k in 1 4; do
  timeout 600 python bench.py --kernel $k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_v_base_k$k.log 2>&1
  W2V_LIBRARY=paper_1611_06172_b200/libw2v_t6.so timeout 600 python bench.py --kernel $k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_v_t6_k$k.log 2>&1
done
