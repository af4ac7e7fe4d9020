# dist tests after the qsv communicator + 32-byte swap; exchange A/B (QSV_SWAP_VEC)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_comm.py -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_dist.txt
for v in 1 0 1 0; do QSV_SWAP_VEC=$v timeout 300 python profiles/time_exchange.py --local 28 >> gpurun_out/xchg_vec$v.txt 2>&1; done
cat gpurun_out/pytest_dist.txt; tail -2 gpurun_out/xchg_vec1.txt | cut -c1-600; tail -2 gpurun_out/xchg_vec0.txt | cut -c1-600
