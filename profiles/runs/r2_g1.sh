set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 600 python profiles/time_jit.py 16 20 24 28 30 > gpurun_out/time_jit.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/time_jit.txt | cut -c1-3000
