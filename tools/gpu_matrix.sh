python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r.log 2>&1
for r in 4 5; do W2V_MIX_PAD=1 timeout 600 python bench.py --kernel 5 --mix-ring-units $r --steps 3 --warmup 2 --no-cpu-baseline --no-rowpath > gpurun_out/mx_r_r$r.log 2>&1; done
