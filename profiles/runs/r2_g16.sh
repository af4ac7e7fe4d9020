# small state: full capture of one generated cnot-ring(16) pass
mkdir -p gpurun_out
python profiles/prof_jit.py cnot-ring 16 2 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 6 -c 1 -o gpurun_out/cnr16_p6 python profiles/prof_jit.py cnot-ring 16 2 > /dev/null 2>&1
ls gpurun_out/cnr16_p6.ncu-rep
