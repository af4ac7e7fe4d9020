# r3 default for n = 12..18 under generated kernels: full GPU suite + small-n timing
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_full44.txt
LS=-1 NS=12,14,16,17,18,19,20 timeout 300 python profiles/time_small_n.py > gpurun_out/sn44.txt 2>&1
cat gpurun_out/pytest_full44.txt gpurun_out/sn44.txt
