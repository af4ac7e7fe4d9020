# static tile assignment for small passes: parity + small-n A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_st.txt
for x in 1 0; do QSV_JIT_STATIC=$x LS=-1,10,11,12 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/st_$x.txt 2>&1; done
cat gpurun_out/pytest_st.txt gpurun_out/st_1.txt gpurun_out/st_0.txt
