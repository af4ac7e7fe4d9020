# warp bits never on local bits 0..3: timing with warp-local transitions on / off
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_wl2.txt
for w in 1 0; do QSV_JIT_WARP_LOCAL=$w timeout 500 python profiles/time_jit.py 24 28 30 > gpurun_out/wl2_$w.txt 2>&1; done
cat gpurun_out/pytest_wl2.txt
