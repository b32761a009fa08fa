python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_s.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ring_det or (cfg1_deterministic and 1)" > gpurun_out/pt_s.log 2>&1; echo "rc $?" >> gpurun_out/pt_s.log
for r in 0 3 5 7 9; do timeout 600 python bench.py --kernel 5 --mix-ring-units $r --steps 3 --warmup 2 --no-cpu-baseline --no-rowpath > gpurun_out/mx_s_r$r.log 2>&1; done
timeout 600 python bench.py --kernel 1 --steps 3 --warmup 2 --no-cpu-baseline --no-rowpath > gpurun_out/mx_s_rows.log 2>&1
