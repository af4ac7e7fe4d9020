# snapshot: full GPU suite + default bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_r2g14.txt
timeout 900 python bench.py > gpurun_out/bench_r2g14.txt 2>&1
tail -3 gpurun_out/pytest_r2g14.txt
