# expectation passes on forked streams: parity + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_expect_jit.py tests/test_gpu_parity.py -m gpu -q -x -k "expect or observable or vqe or cfg3 or tfim" 2>&1 | tail -2 > gpurun_out/pytest_lanes.txt
for x in 3 1 3 1; do echo "# lanes $x"; QSV_EXPECT_STREAMS=$x timeout 300 python profiles/time_expect_jit.py 20 22 24 26 28 2>&1 | grep -v "^{" | python -c "
import sys, json
for l in sys.stdin:
    n, j = l.split(' ', 1); d = json.loads(j)
    print(n, 'device %.4f ms' % (d['device_s']*1e3), 'wall %.4f ms' % (d['wall_s']*1e3), 'hbm_frac %.2f' % d['hbm_frac'])
"; done > gpurun_out/lanes_ab.txt
cat gpurun_out/pytest_lanes.txt gpurun_out/lanes_ab.txt
