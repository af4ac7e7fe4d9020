# late griddepcontrol.wait (static, direct-load passes): parity + small-n A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_lw.txt
for x in 1 0 1 0; do echo "# LATE_WAIT=$x"; QSV_JIT_LATE_WAIT=$x LS=-1 NS=12,14,16,17,18 timeout 300 python profiles/time_small_n.py; done > gpurun_out/lw.txt 2>&1
cat gpurun_out/pytest_lw.txt gpurun_out/lw.txt
