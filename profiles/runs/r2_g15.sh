# DMMA dense-5 kernel: parity (dense K=1..8 + heavy(5) golden) and A/B vs the DFMA kernel + ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or golden or heavy or circuit" 2>&1 | tail -4 > gpurun_out/pytest_mma.txt
for m in 1 0; do for n in 20 28 30; do QSV_DENSE5_MMA=$m timeout 120 python profiles/time_dense5.py $n >> gpurun_out/dense5_$m.txt 2>&1; done; done
QSV_DENSE5_MMA=1 timeout 120 python profiles/time_dense5.py 28 0 1 2 3 4 >> gpurun_out/dense5_1.txt 2>&1
QSV_DENSE5_MMA=0 timeout 120 python profiles/time_dense5.py 28 0 1 2 3 4 >> gpurun_out/dense5_0.txt 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_dense5 -s 1 -c 1 -o gpurun_out/dense5_mma env QSV_DENSE5_MMA=1 python profiles/time_dense5.py 28 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:k_dense5 -s 1 -c 1 -o gpurun_out/dense5_dfma env QSV_DENSE5_MMA=0 python profiles/time_dense5.py 28 > /dev/null 2>&1
cat gpurun_out/pytest_mma.txt gpurun_out/dense5_1.txt gpurun_out/dense5_0.txt
