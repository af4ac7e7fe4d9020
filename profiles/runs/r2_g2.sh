# full GPU suite + ncu of one generated pass kernel (cz-ladder / cnot-ring n=28)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1   # fills the JIT disk cache
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 3 -c 1 -o gpurun_out/jit_czl28 python profiles/prof_jit.py cz-ladder 28 2 > gpurun_out/ncu_czl.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 5 -c 1 -o gpurun_out/jit_cnr28 python profiles/prof_jit.py cnot-ring 28 2 > gpurun_out/ncu_cnr.log 2>&1
tail -3 gpurun_out/pytest_gpu.txt
