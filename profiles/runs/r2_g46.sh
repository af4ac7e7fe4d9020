# small-n: PDL A/B with static tiles + r3
mkdir -p gpurun_out
for x in 0 1 0 1; do QSV_PDL=$x LS=-1 NS=12,14,16,18,20 timeout 300 python profiles/time_small_n.py > gpurun_out/pdl46_$x.txt 2>&1; cat gpurun_out/pdl46_$x.txt; done
