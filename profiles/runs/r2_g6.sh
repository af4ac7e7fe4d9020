# small states: programmatic dependent launch A/B, tile size sweep (generated passes)
mkdir -p gpurun_out
for pdl in 1 0; do QSV_PDL=$pdl LS=-1,9,10,11,12 timeout 600 python profiles/time_small_n.py > gpurun_out/small_pdl$pdl.txt 2>&1; done
cat gpurun_out/small_pdl1.txt gpurun_out/small_pdl0.txt
