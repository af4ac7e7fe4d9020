# expectation: register-staged loads A/B + parity
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_expect_jit.py tests/test_gpu_parity.py -m gpu -q -x -k "expect or observable or tfim or vqe or golden" 2>&1 | tail -2 > gpurun_out/pytest_rl.txt
for r in 1 0 1 0; do QSV_EXPECT_REGLOAD=$r timeout 300 python profiles/time_expect_jit.py 24 26 28 >> gpurun_out/texp_rl$r.txt 2>&1; done
cat gpurun_out/pytest_rl.txt
