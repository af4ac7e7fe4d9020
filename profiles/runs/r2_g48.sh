# single-launch programs: spin barrier (no nanosleep) timing A/B
mkdir -p gpurun_out
for x in 1 0; do QSV_MEGA=$x LS=-1 NS=12,14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega48_$x.txt 2>&1; done
cat gpurun_out/mega48_1.txt gpurun_out/mega48_0.txt
