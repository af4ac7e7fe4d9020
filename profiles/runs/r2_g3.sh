# expectation JIT: tests + timing (jit vs generic); tile JIT variant A/B for cz-ladder
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_expect_jit.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_r2g3.txt
QSV_EXPECT_JIT=0 timeout 300 python profiles/time_expect_jit.py 24 28 > gpurun_out/texp_generic.txt 2>&1
timeout 300 python profiles/time_expect_jit.py 24 28 > gpurun_out/texp_jit.txt 2>&1
for v in 4 5; do QSV_TILE_VARIANT=$v timeout 300 python profiles/time_jit.py 28 30 > gpurun_out/tjit_v$v.txt 2>&1; done
tail -3 gpurun_out/pytest_r2g3.txt; tail -1 gpurun_out/texp_generic.txt; tail -1 gpurun_out/texp_jit.txt
