# timing bounds: group barriers -> warp barriers (1), transitions without shared memory (2)
mkdir -p gpurun_out
for x in 0 1 2; do QSV_JIT_EXPERIMENT=$x timeout 500 python profiles/time_jit.py 24 28 30 > gpurun_out/exp_$x.txt 2>&1; done
