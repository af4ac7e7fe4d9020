# single-launch programs: cooperative vs plain launch cost (probe; plain launch is not co-residency safe)
mkdir -p gpurun_out
QSV_MEGA_COOP=0 QSV_MEGA_EMPTY=1 LS=-1 NS=14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega50_empty_plain.txt 2>&1
QSV_MEGA_COOP=0 LS=-1 NS=14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega50_plain.txt 2>&1
QSV_MEGA=0 LS=-1 NS=14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega50_off.txt 2>&1
cat gpurun_out/mega50_empty_plain.txt gpurun_out/mega50_plain.txt gpurun_out/mega50_off.txt
