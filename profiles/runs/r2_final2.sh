# late-round snapshot: full GPU suite, smoke, bench, launch list, small-state tile sweep for r3
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final3_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.txt 2>&1
( time timeout 900 python bench.py > gpurun_out/final3_bench.txt 2>&1 ) 2> gpurun_out/final3_bench_time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/final3_bench_launches.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
QSV_TILE_VARIANT=3 LS=8,9,10,11 NS=12,14,16 timeout 300 python profiles/time_small_n.py > gpurun_out/final3_r3_tiles.txt 2>&1
cat gpurun_out/final3_pytest.txt gpurun_out/final3_smoke.txt gpurun_out/final3_bench_time.txt gpurun_out/final3_r3_tiles.txt
