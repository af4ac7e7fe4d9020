# single-launch programs: placement probe (1 CTA/SM) and barrier-only cost
mkdir -p gpurun_out
QSV_MEGA_SMEM=120000 LS=-1 NS=14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega49_smem.txt 2>&1
QSV_MEGA_EMPTY=1 LS=-1 NS=14,16,18 timeout 300 python profiles/time_small_n.py > gpurun_out/mega49_empty.txt 2>&1
cat gpurun_out/mega49_smem.txt gpurun_out/mega49_empty.txt
