# one-FMA rotations: parity + timing A/B (variant x one_fma)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_r2g4.txt
for f in 1 0; do for v in 4 5; do QSV_ONE_FMA=$f QSV_TILE_VARIANT=$v timeout 300 python profiles/time_jit.py 20 28 30 > gpurun_out/tjit_f${f}_v$v.txt 2>&1; done; done
tail -3 gpurun_out/pytest_r2g4.txt
