# shuffle transitions: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_sh.txt
for x in 1 0; do QSV_JIT_SHUFFLE=$x timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/sh_$x.txt 2>&1; done
QSV_JIT_SHUFFLE=1 LS=-1 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/sh_small.txt 2>&1
cat gpurun_out/pytest_sh.txt
