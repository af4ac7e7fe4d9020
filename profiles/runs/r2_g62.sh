# extended planner fuzz: 600 random circuits / plan options / variants (incl. r3, auto tiles) vs the C oracle
mkdir -p gpurun_out
QSV_FUZZ_CASES=600 timeout 3000 python -m pytest tests/test_gpu_tiles.py -m gpu -q -x -k fuzz 2>&1 | tail -3 > gpurun_out/fuzz600.txt
cat gpurun_out/fuzz600.txt
