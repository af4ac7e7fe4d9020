# r3 after the smem-limit fix: parity + small-state timing; new default (r4 under JIT)
mkdir -p gpurun_out
QSV_TILE_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x -k "tiles or circuit or golden" 2>&1 | tail -4 > gpurun_out/pytest_r3.txt
QSV_TILE_VARIANT=3 LS=-1,10,11,12 NS=14,16,18,20,22 timeout 600 python profiles/time_small_n.py > gpurun_out/small_v3.txt 2>&1
LS=-1 NS=14,16,18,20,22 timeout 600 python profiles/time_small_n.py > gpurun_out/small_def2.txt 2>&1
timeout 300 python profiles/time_jit.py 28 30 > gpurun_out/tjit_def2.txt 2>&1
cat gpurun_out/pytest_r3.txt gpurun_out/small_v3.txt gpurun_out/small_def2.txt; grep -v "^{" gpurun_out/tjit_def2.txt | cut -c1-200
