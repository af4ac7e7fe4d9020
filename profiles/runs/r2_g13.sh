# phase cap per pass (instruction-cache footprint vs number of passes)
mkdir -p gpurun_out
for c in 1000 12 10 8 6; do QSV_MAX_PASS_PHASES=$c timeout 400 python profiles/time_jit.py 24 28 30 > gpurun_out/cap_$c.txt 2>&1; done
for c in 1000 12 10 8 6; do echo "cap=$c"; grep -v "^{\"cz\|jit_stats" gpurun_out/cap_$c.txt | cut -c1-30; done
