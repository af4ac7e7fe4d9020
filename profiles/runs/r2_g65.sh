# planner fuzz with two more seeds (400 cases each) after per-program PDL and expectation lanes
mkdir -p gpurun_out
for seed in 7 99; do QSV_FUZZ_SEED=$seed QSV_FUZZ_CASES=400 timeout 1500 python -m pytest tests/test_gpu_tiles.py -m gpu -q -x -k fuzz 2>&1 | tail -1; done > gpurun_out/fuzz_seeds.txt
cat gpurun_out/fuzz_seeds.txt
