# physical DRAM traffic of CZ / CNOT per target (ncu)
mkdir -p gpurun_out
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_diag|k_pair2x2" --csv python profiles/dram_per_target.py > gpurun_out/dram_per_target.csv 2>&1
tail -3 gpurun_out/dram_per_target.csv
