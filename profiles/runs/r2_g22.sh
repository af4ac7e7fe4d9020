# warp-local phase transitions (QSV_JIT_WARP_LOCAL) + maps / density tests after the rewrite
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_maps.py tests/test_density.py tests/test_serialize_cli.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_wl.txt
for w in 1 0; do QSV_JIT_WARP_LOCAL=$w timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/wl_$w.txt 2>&1; done
for w in 1 0; do QSV_JIT_WARP_LOCAL=$w LS=-1 NS=14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/wl_small_$w.txt 2>&1; done
cat gpurun_out/pytest_wl.txt
