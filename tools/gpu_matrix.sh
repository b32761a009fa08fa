python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_o.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x -k "prefetch or host_pointer or replicas or nccl_one_rank" > gpurun_out/pt_o.log 2>&1; echo "rc $?" >> gpurun_out/pt_o.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/mx_o.log 2>&1
