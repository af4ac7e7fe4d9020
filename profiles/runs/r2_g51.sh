# single-launch programs: constant-block copy cost probe
mkdir -p gpurun_out
QSV_MEGA_NOCOPY=1 QSV_MEGA_EMPTY=1 LS=-1 NS=16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega51_empty_nocopy.txt 2>&1
QSV_MEGA_NOCOPY=1 LS=-1 NS=16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega51_nocopy.txt 2>&1
cat gpurun_out/mega51_empty_nocopy.txt gpurun_out/mega51_nocopy.txt
