# end-of-round snapshot: full GPU suite, smoke, bench, VQE iteration probe
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/final7_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 > gpurun_out/final7_smoke.txt
( time timeout 900 python bench.py > gpurun_out/final7_bench.txt 2>&1 ) 2> gpurun_out/final7_bench_time.txt
timeout 300 python profiles/time_vqe_iter.py > gpurun_out/final7_vqe_iter.txt 2>&1
cat gpurun_out/final7_pytest.txt gpurun_out/final7_smoke.txt gpurun_out/final7_bench_time.txt; tail -5 gpurun_out/final7_vqe_iter.txt
