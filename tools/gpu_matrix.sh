# tools/gpu_matrix.sh — one gpurun session of timing experiments + ncu captures (round 2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_g.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "mode2 or (cfg1_deterministic and 1)" > gpurun_out/pt_g.log 2>&1; echo "rc $?" >> gpurun_out/pt_g.log
for spec in "3 1" "4 1" "3 4"; do set -- $spec
  timeout 300 python bench.py --config $1 --kernel $2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_g_c$1_k$2.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hogbatch_step -s 2 -c 1 -o gpurun_out/prof_cfg4_r02b python bench.py --config 4 --kernel 1 --tokens 134216000 --steps 1 --warmup 1 --no-cpu-baseline --no-rowpath > gpurun_out/ncu_cfg4b.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hogbatch_step -s 2 -c 1 -o gpurun_out/prof_cfg3_r02 python bench.py --config 3 --kernel 1 --tokens 134217720 --steps 1 --warmup 1 --no-cpu-baseline --no-rowpath > gpurun_out/ncu_cfg3.log 2>&1
