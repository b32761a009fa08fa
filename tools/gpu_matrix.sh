python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_u.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "cfg4 or edge or mode2 or cfg1_deterministic" > gpurun_out/pt_u.log 2>&1; echo "rc $?" >> gpurun_out/pt_u.log
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_u_cfg4.log 2>&1
