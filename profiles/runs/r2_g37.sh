# sharded path with generated pass kernels (jit=2 for shard programs)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_dist2.txt
timeout 900 python bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded2.txt 2>&1
cat gpurun_out/pytest_dist2.txt
