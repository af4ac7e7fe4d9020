# small-n: per-pass kernel durations (warm L2) vs event-timed circuit, r3 default
mkdir -p gpurun_out
python profiles/small_n_launches.py > gpurun_out/sn45_plain.txt 2>&1
RUNS=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.max --cache-control none --clock-control none --csv --log-file gpurun_out/sn45_launches.csv python profiles/small_n_launches.py > gpurun_out/sn45_ncu.txt 2>&1
