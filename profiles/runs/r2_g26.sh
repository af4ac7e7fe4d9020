# full suite after the source cache + bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_r2g26.txt
timeout 900 python bench.py > gpurun_out/bench_r2g26.txt 2>&1
cat gpurun_out/pytest_r2g26.txt
