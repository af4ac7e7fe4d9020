# multi-start tile-set selection: parity + timing A/B (QSV_PASS_SEARCH)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_jit.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_search.txt
for s in 1 0; do QSV_PASS_SEARCH=$s timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/search_$s.txt 2>&1; done
for s in 1 0; do QSV_PASS_SEARCH=$s LS=-1 NS=14,16,18,20,22 timeout 300 python profiles/time_small_n.py > gpurun_out/search_small_$s.txt 2>&1; done
cat gpurun_out/pytest_search.txt
