# generated passes: next tile prefetched as soon as the buffer is free + direct store from the last phase (A/B)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py -m gpu -q -x 2>&1 | tail -4 > gpurun_out/pytest_direct.txt
for d in 1 0; do QSV_JIT_DIRECT_STORE=$d timeout 400 python profiles/time_jit.py 20 24 28 30 > gpurun_out/direct_$d.txt 2>&1; done
cat gpurun_out/pytest_direct.txt
for d in 1 0; do echo "direct=$d"; grep -v "^{\"cz\|jit_stats" gpurun_out/direct_$d.txt | cut -c1-40; done
