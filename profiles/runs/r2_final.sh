# final snapshot of round 2: suite, smoke, bench, launch list, captures of the hot kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/final_bench.txt 2>&1 ) 2> gpurun_out/final_bench_time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/final_bench_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 0 -c 1 -o gpurun_out/final2_czl28_p0 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 8 -c 1 -o gpurun_out/final2_czl28_p8 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_pass --csv python profiles/prof_jit.py cz-ladder 28 2 > gpurun_out/final2_czl28_launches.csv 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_pass -s 4 -c 1 -o gpurun_out/final2_expect_n28 python profiles/time_expect_jit.py 28 > /dev/null 2>&1
cat gpurun_out/final_pytest.txt gpurun_out/final_smoke.txt gpurun_out/final_bench_time.txt
