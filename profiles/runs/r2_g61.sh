# expectation (TFIM) wall vs device time at n = 20..28, plus kernel launch list at n = 24
mkdir -p gpurun_out
timeout 300 python profiles/time_expect_jit.py 20 22 24 26 28 > gpurun_out/exp61.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/exp61_launches.csv python profiles/time_expect_jit.py 24 > /dev/null 2>&1
grep -v "^{" gpurun_out/exp61.txt | cut -c1-400
