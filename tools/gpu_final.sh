# tools/gpu_final.sh — round-2 evidence session: full GPU suite, smoke, default bench (driver's
# K/W), launch list + ncu --set full of the step kernel, the other configs' bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fin2.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s --durations=25 > gpurun_out/pt_fin2.log 2>&1; echo "pytest rc $?" >> gpurun_out/pt_fin2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_fin2.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_fin2.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_fin2.log 2>&1; echo "bench rc $?" >> gpurun_out/bench_fin2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_fin2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_fin2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hogbatch_step -s 2 -c 1 -o gpurun_out/prof_fin2 python bench.py --tokens 134217720 --steps 1 --warmup 1 --no-cpu-baseline --no-rowpath > gpurun_out/ncu_fin2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hogbatch_step -s 2 -c 1 -o gpurun_out/prof_cfg4_fin2 python bench.py --config 4 --tokens 134216000 --steps 1 --warmup 1 --no-cpu-baseline --no-rowpath > gpurun_out/ncu_cfg4_fin2.log 2>&1
timeout 900 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_fin2_cfg4.log 2>&1
timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_fin2_cfg5.log 2>&1
timeout 900 python bench.py --algorithm alg1 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_fin2_alg1.log 2>&1
timeout 900 python bench.py --kernel 4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_fin2_ring.log 2>&1
timeout 600 python tools/sanitize_run.py > gpurun_out/sanitize_fin2.log 2>&1; echo "sanitize rc $?" >> gpurun_out/sanitize_fin2.log
