# direct load with the strict (lanes = qubits 0..3) direct store
mkdir -p gpurun_out
QSV_JIT_DIRECT_LOAD=1 QSV_JIT_DIRECT_ANY=0 timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/dl_10.txt 2>&1
QSV_JIT_DIRECT_LOAD=1 QSV_JIT_DIRECT_ANY=1 timeout 500 python profiles/time_jit.py 20 24 28 30 > gpurun_out/dl_11b.txt 2>&1
