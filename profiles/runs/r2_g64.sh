# automatic PDL for shallow small programs: parity + A/B vs off
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_apdl.txt
for x in auto 0 auto 0; do echo "# QSV_PDL=$x"; if [ $x = auto ]; then LS=-1 NS=12,14,16,17,18,19,20,22 timeout 300 python profiles/time_small_n.py; else QSV_PDL=0 LS=-1 NS=12,14,16,17,18,19,20,22 timeout 300 python profiles/time_small_n.py; fi; done > gpurun_out/apdl.txt 2>&1
cat gpurun_out/pytest_apdl.txt gpurun_out/apdl.txt
