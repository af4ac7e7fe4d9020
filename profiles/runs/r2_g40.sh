# small-n: per-pass kernel durations vs event-timed circuit; r5 vs r4 on large n
mkdir -p gpurun_out
python profiles/small_n_launches.py > gpurun_out/sn_plain.txt 2>&1
RUNS=3 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/sn_launches.csv python profiles/small_n_launches.py > gpurun_out/sn_ncu.txt 2>&1
for v in 5; do QSV_TILE_VARIANT=$v timeout 500 python profiles/time_jit.py 24 28 30 > gpurun_out/var_$v.txt 2>&1; done
