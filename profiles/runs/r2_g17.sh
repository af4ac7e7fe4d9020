# 8-amplitude (r3) tile variant: parity + small-state timing vs r4 / default
mkdir -p gpurun_out
QSV_TILE_VARIANT=3 timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x -k "tiles or circuit or golden" 2>&1 | tail -4 > gpurun_out/pytest_r3.txt
for v in 3 4; do QSV_TILE_VARIANT=$v LS=-1,10,11,12 NS=14,16,18,20,22 timeout 600 python profiles/time_small_n.py > gpurun_out/small_v$v.txt 2>&1; done
LS=-1 NS=14,16,18,20,22 timeout 600 python profiles/time_small_n.py > gpurun_out/small_def.txt 2>&1
cat gpurun_out/pytest_r3.txt gpurun_out/small_v3.txt gpurun_out/small_v4.txt gpurun_out/small_def.txt
