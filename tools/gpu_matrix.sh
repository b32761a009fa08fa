# tools/gpu_matrix.sh — one gpurun session of timing experiments (round 2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_h.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mode2 or (cfg1_deterministic and 1) or (edge and 1) or cfg4_full or (cfg1_hogwild and 1) or ring_det" > gpurun_out/pt_h.log 2>&1; echo "rc $?" >> gpurun_out/pt_h.log
for spec in "4 1" "3 1"; do set -- $spec
  timeout 300 python bench.py --config $1 --kernel $2 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_h_c$1_k$2.log 2>&1
done
