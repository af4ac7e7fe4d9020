# late sync (barrier + next-tile publication after the HBM loads): parity + A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_ls.txt
for x in 1 0; do QSV_JIT_LATE_SYNC=$x timeout 500 python profiles/time_jit.py 24 28 30 > gpurun_out/ls_$x.txt 2>&1; done
for x in 1 0; do QSV_JIT_LATE_SYNC=$x LS=-1 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/ls_small_$x.txt 2>&1; done
cat gpurun_out/pytest_ls.txt gpurun_out/ls_small_1.txt gpurun_out/ls_small_0.txt
