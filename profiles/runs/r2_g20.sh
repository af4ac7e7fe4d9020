# tile-set search with one pass of lookahead (QSV_PASS_SEARCH=2) vs multi-start (1)
mkdir -p gpurun_out
QSV_PASS_SEARCH=2 timeout 900 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_jit.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_search2.txt
for s in 2 1; do QSV_PASS_SEARCH=$s timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/search2_$s.txt 2>&1; done
QSV_PASS_SEARCH=2 LS=-1 NS=14,16,18,20,22 timeout 300 python profiles/time_small_n.py > gpurun_out/search_small_2.txt 2>&1
cat gpurun_out/pytest_search2.txt
