# single-launch programs (cooperative megakernel) for small states: parity + timing A/B
mkdir -p gpurun_out
QSV_JIT_VERBOSE=1 timeout 600 python profiles/small_n_launches.py > gpurun_out/mega_probe.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_mega.txt
for x in 1 0; do QSV_MEGA=$x LS=-1 NS=12,14,16,17,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega_$x.txt 2>&1; done
cat gpurun_out/mega_probe.txt gpurun_out/pytest_mega.txt gpurun_out/mega_1.txt gpurun_out/mega_0.txt
