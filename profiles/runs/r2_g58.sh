# r3 on 12-qubit tiles (512-thread groups, one per CTA, generated kernels only): parity + timing
mkdir -p gpurun_out
QSV_TILE_VARIANT=3 timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x -k "not n30 and not cfg4" 2>&1 | tail -3 > gpurun_out/pytest_r3l12.txt
echo "# r3 L=12" > gpurun_out/r3l12.txt
QSV_TILE_VARIANT=3 LS=12 NS=16,18,19,20,21,22,24 timeout 400 python profiles/time_small_n.py >> gpurun_out/r3l12.txt 2>&1
echo "# default" >> gpurun_out/r3l12.txt
LS=-1 NS=16,18,19,20,21,22,24 timeout 400 python profiles/time_small_n.py >> gpurun_out/r3l12.txt 2>&1
cat gpurun_out/pytest_r3l12.txt gpurun_out/r3l12.txt
