mkdir -p gpurun_out
K='regex:sor_pass_tma<\(int\)0, \(bool\)0, \(bool\)0, \(bool\)1>'
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base --kernel-name-base demangled -k "$K" -s 5 -c 3 --csv python scripts/sweep_rate.py config1 > gpurun_out/clk_base.csv 2> gpurun_out/clk_base.err
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k "$K" -s 5 -c 3 --csv python scripts/sweep_rate.py config1 > gpurun_out/clk_none.csv 2> gpurun_out/clk_none.err
nvidia-smi -q -d CLOCK > gpurun_out/clocks.txt
