# single-launch programs: kernel durations under ncu (empty barrier chain / full)
mkdir -p gpurun_out
QSV_MEGA_EMPTY=1 RUNS=3 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__cycles_active.max --cache-control none --clock-control none --csv --log-file gpurun_out/mega52_empty.csv python profiles/small_n_launches.py > gpurun_out/mega52_e.txt 2>&1
RUNS=3 timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__cycles_active.max --cache-control none --clock-control none --csv --log-file gpurun_out/mega52_full.csv python profiles/small_n_launches.py > gpurun_out/mega52_f.txt 2>&1
