python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg1_deterministic or edge or mode2 or ring_det or cfg4_shape or cfg1_hogwild" > gpurun_out/pt_t.log 2>&1; echo "rc $?" >> gpurun_out/pt_t.log
for c in 3 4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/mx_t_cfg$c.log 2>&1; done
