# cz-ladder(28) generated passes after one-FMA: launch list (per-pass time + DRAM) and full captures of a heavy and a light pass
mkdir -p gpurun_out
python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_pass --csv python profiles/prof_jit.py cz-ladder 28 2 > gpurun_out/czl28_launches.csv 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 0 -c 1 -o gpurun_out/czl28_p0 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 14 -c 1 -o gpurun_out/czl28_p14 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
ls gpurun_out
