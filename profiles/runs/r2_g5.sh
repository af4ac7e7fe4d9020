# full GPU suite after one-FMA + launch caching; bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_r2g5.txt
timeout 600 python bench.py > gpurun_out/bench_r2g5.txt 2>&1
tail -3 gpurun_out/pytest_r2g5.txt
