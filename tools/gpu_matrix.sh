# tools/gpu_matrix.sh — one gpurun session of checks + timings (round 2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_l.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_alg1.py -q -s -k "cfg4 or edge or cfg1 or mode2 or ring_det or ring_delta or host_pointer or checkpoint or headline" > gpurun_out/pt_l.log 2>&1; echo "rc $?" >> gpurun_out/pt_l.log
for k in 1 4; do timeout 600 python bench.py --kernel $k --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_l_k$k.log 2>&1; done
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_l_cfg4.log 2>&1
