# snapshot 4: full suite + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_r2g32.txt
( time timeout 900 python bench.py > gpurun_out/bench_r2g32.txt 2>&1 ) 2> gpurun_out/bench_r2g32_time.txt
cat gpurun_out/pytest_r2g32.txt gpurun_out/bench_r2g32_time.txt
