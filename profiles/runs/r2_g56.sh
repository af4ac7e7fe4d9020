# planner fuzz with the 8-amplitude variant and auto tile sizes (200 cases) + the suite's 40
mkdir -p gpurun_out
QSV_FUZZ_CASES=200 timeout 1500 python -m pytest tests/test_gpu_tiles.py -m gpu -q -x -k fuzz 2>&1 | tail -3 > gpurun_out/fuzz200.txt
cat gpurun_out/fuzz200.txt
