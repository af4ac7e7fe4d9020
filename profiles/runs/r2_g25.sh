# no-hoist A/B + jit/tiles parity
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_nh.txt
for h in 1 0; do QSV_JIT_NOHOIST=$h timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/nh_$h.txt 2>&1; done
cat gpurun_out/pytest_nh.txt
