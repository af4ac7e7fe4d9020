# small-n: one full ncu capture of a mid-circuit cnot-ring(16) pass
mkdir -p gpurun_out
RUNS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass --launch-skip 24 --launch-count 1 -o gpurun_out/sn_pass python profiles/small_n_launches.py > gpurun_out/sn_full.txt 2>&1
