# snapshot after slot addressing / static tiles / r3: smoke, bench, launch list, pass-8 capture
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g53_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/g53_bench.txt 2>&1 ) 2> gpurun_out/g53_bench_time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/g53_bench_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_pass -s 8 -c 1 -o gpurun_out/g53_czl28_p8 python profiles/prof_jit.py cz-ladder 28 2 > /dev/null 2>&1
cat gpurun_out/g53_smoke.txt gpurun_out/g53_bench_time.txt
