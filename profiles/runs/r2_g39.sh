# split slot addresses + folded sign xors: parity + A/B; call overhead probe
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_as.txt
for x in 1 0; do QSV_JIT_ADDR_SPLIT=$x QSV_JIT_SIGN_FOLD=$x timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/as_$x.txt 2>&1; done
QSV_JIT_ADDR_SPLIT=1 QSV_JIT_SIGN_FOLD=0 timeout 500 python profiles/time_jit.py 28 30 > gpurun_out/as_10.txt 2>&1
timeout 300 python profiles/time_call_overhead.py > gpurun_out/call_overhead.txt 2>&1
cat gpurun_out/pytest_as.txt
