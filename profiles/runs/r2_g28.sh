# direct first-phase loads / relaxed direct stores: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_dl.txt
QSV_JIT_DIRECT_LOAD=1 QSV_JIT_DIRECT_ANY=1 timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/dl_11.txt 2>&1
QSV_JIT_DIRECT_LOAD=0 QSV_JIT_DIRECT_ANY=1 timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/dl_01.txt 2>&1
QSV_JIT_DIRECT_LOAD=0 QSV_JIT_DIRECT_ANY=0 timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/dl_00.txt 2>&1
QSV_JIT_DIRECT_LOAD=1 LS=-1 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/dl_small_1.txt 2>&1
QSV_JIT_DIRECT_LOAD=0 QSV_JIT_DIRECT_ANY=0 LS=-1 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/dl_small_0.txt 2>&1
cat gpurun_out/pytest_dl.txt
