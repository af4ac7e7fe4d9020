# small-n (r3, static tiles): full ncu capture of one mid-circuit cnot-ring(16) pass
mkdir -p gpurun_out
RUNS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pass --launch-skip 30 --launch-count 1 -o gpurun_out/sn_r3_pass python profiles/small_n_launches.py > gpurun_out/sn_r3_full.txt 2>&1
