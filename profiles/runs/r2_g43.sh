# r3 (8 amplitudes per thread) under generated kernels: parity + small-n timing
mkdir -p gpurun_out
QSV_TILE_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x -k "not n30 and not cfg4" 2>&1 | tail -4 > gpurun_out/pytest_r3.txt
QSV_TILE_VARIANT=3 LS=-1,10,11 NS=12,14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/r3_small.txt 2>&1
LS=-1,10,11,12 NS=12,14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/r4_small.txt 2>&1
cat gpurun_out/pytest_r3.txt gpurun_out/r3_small.txt gpurun_out/r4_small.txt
