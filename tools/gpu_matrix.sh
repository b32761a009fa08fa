python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_p.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_alg1.py -q -s -k "cfg4 or edge or cfg1 or mode2 or ring_det or host_pointer or checkpoint or prefetch" > gpurun_out/pt_p.log 2>&1; echo "rc $?" >> gpurun_out/pt_p.log
for c in 4 3; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_p_cfg$c.log 2>&1; done
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline --no-rowpath > gpurun_out/mx_p_cfg5.log 2>&1
