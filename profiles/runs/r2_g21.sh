# snapshot 2: full GPU suite + default bench + time_jit
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/pytest_r2g21.txt
timeout 900 python bench.py > gpurun_out/bench_r2g21.txt 2>&1
timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/tjit_r2g21.txt 2>&1
tail -3 gpurun_out/pytest_r2g21.txt
