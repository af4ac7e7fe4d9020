# variant A/B after direct loads
mkdir -p gpurun_out
for v in 5 4; do QSV_TILE_VARIANT=$v timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/var_$v.txt 2>&1; done
