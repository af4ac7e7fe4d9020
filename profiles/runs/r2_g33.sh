# expectation regload with streaming loads (LDG.E.EF) vs cp.async
mkdir -p gpurun_out
for r in 1 0 1 0; do QSV_EXPECT_REGLOAD=$r timeout 300 python profiles/time_expect_jit.py 24 26 28 >> gpurun_out/texp_rlef$r.txt 2>&1; done
QSV_EXPECT_REGLOAD=1 timeout 300 python -m pytest tests/test_expect_jit.py -m gpu -q 2>&1 | tail -2
