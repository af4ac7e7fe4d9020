# expectation passes: cp.async (16 B) vs cp.async.bulk (256 B runs + mbarrier) A/B + parity
mkdir -p gpurun_out
QSV_EXPECT_BULK=1 timeout 600 python -m pytest tests/test_expect_jit.py -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_bulk.txt
for b in 0 1 0 1; do QSV_EXPECT_BULK=$b timeout 300 python profiles/time_expect_jit.py 24 26 28 >> gpurun_out/texp_bulk$b.txt 2>&1; done
timeout 300 ncu --set full --clock-control none -k regex:k_pass -s 4 -c 1 -o gpurun_out/xbulk0_n28 env QSV_EXPECT_BULK=0 python profiles/time_expect_jit.py 28 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_pass -s 4 -c 1 -o gpurun_out/xbulk1_n28 env QSV_EXPECT_BULK=1 python profiles/time_expect_jit.py 28 > /dev/null 2>&1
cat gpurun_out/pytest_bulk.txt; grep -h '^{' gpurun_out/texp_bulk0.txt gpurun_out/texp_bulk1.txt | cut -c1-400
