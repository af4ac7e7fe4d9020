# sharded path on one GPU (4 virtual ranks) with the round-2 kernels
mkdir -p gpurun_out
timeout 900 python bench.py --sharded --steps 3 --warmup 3 > gpurun_out/bench_sharded.txt 2>&1
tail -c 3000 gpurun_out/bench_sharded.txt
