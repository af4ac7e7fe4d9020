# group stagger vs lockstep for deep generated passes (instruction-cache sharing)
mkdir -p gpurun_out
for t in 1000 12 6 0; do QSV_STAGGER_MAX_PHASES=$t timeout 300 python profiles/time_jit.py 28 30 > gpurun_out/stag_$t.txt 2>&1; done
for t in 1000 12 6 0; do echo "max_phases=$t"; grep -v "^{\|jit_stats" gpurun_out/stag_$t.txt | cut -c1-60; done
