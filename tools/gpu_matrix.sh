# tools/gpu_matrix.sh — gather engines + L2 cap counters (round 2)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_i.log 2>&1
timeout 300 python tools/engines.py 12 11 > gpurun_out/engines_r02.json 2> gpurun_out/engines_r02.err
timeout 300 python tools/caps.py 1200 11 11 > gpurun_out/caps_r02.json 2> gpurun_out/caps_r02.err
M=lts__t_sectors.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_red.sum,lts__cycles_elapsed.avg,gpu__time_duration.sum,lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_ltcfabric.sum,l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:engine_kernel python tools/engines.py 12 11 > gpurun_out/engines_ncu.csv 2> gpurun_out/engines_ncu.err
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:rowpath_kernel python tools/caps.py 1200 11 11 > gpurun_out/caps_ncu.csv 2> gpurun_out/caps_ncu.err
