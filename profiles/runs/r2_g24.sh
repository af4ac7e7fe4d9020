# snapshot 3: full suite, bench wall time, bench launch list, final k_pass captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_r2g24.txt
( time timeout 900 python bench.py > gpurun_out/bench_r2g24.txt 2>&1 ) 2> gpurun_out/bench_r2g24_time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 0 -c 1 -o gpurun_out/final_czl28_p0 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 8 -c 1 -o gpurun_out/final_czl28_p8 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_pass --csv python profiles/prof_jit.py cz-ladder 28 2 > gpurun_out/final_czl28_launches.csv 2>&1
cat gpurun_out/pytest_r2g24.txt gpurun_out/bench_r2g24_time.txt
