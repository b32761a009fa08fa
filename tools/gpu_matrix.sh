# tools/gpu_matrix.sh — one gpurun session of kernel/config timing experiments (round 2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_f.log 2>&1
python -c "
import sys; sys.path.insert(0, '.')
from paper_1611_06172_b200 import _build
_build.build(out='paper_1611_06172_b200/libw2v_pair8.so', extra=['-DW2V_PAIR_MINB=8'])" >> gpurun_out/build_f.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "(cfg1_deterministic and 5) or (edge and 5) or (cfg1_hogwild and 5)" > gpurun_out/pt_pair.log 2>&1; echo "rc $?" >> gpurun_out/pt_pair.log
for spec in "4 1" "4 5" "3 5"; do set -- $spec
  timeout 300 python bench.py --config $1 --kernel $2 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mx_c$1_k$2.log 2>&1
done
W2V_LIBRARY=paper_1611_06172_b200/libw2v_pair8.so timeout 300 python bench.py --config 4 --kernel 5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/mx_c4_k5_minb8.log 2>&1
