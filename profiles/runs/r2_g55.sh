# PDL trigger placement A/B (off / at kernel start / after the CTA's last tile)
mkdir -p gpurun_out
QSV_PDL=1 QSV_PDL_LATE=1 timeout 900 python -m pytest tests/test_gpu_jit.py tests/test_gpu_tiles.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_pdl.txt
for cfg in "0 0" "1 0" "1 1" "0 0" "1 1"; do set -- $cfg; echo "# PDL=$1 LATE=$2"; QSV_PDL=$1 QSV_PDL_LATE=$2 LS=-1 NS=12,14,16,18,20,22 timeout 300 python profiles/time_small_n.py 2>&1; done > gpurun_out/pdl55.txt
for cfg in "0 0" "1 1"; do set -- $cfg; echo "# PDL=$1 LATE=$2"; QSV_PDL=$1 QSV_PDL_LATE=$2 timeout 500 python profiles/time_jit.py 24 28 2>&1 | grep -v "^{"; done > gpurun_out/pdl55_big.txt
cat gpurun_out/pytest_pdl.txt gpurun_out/pdl55.txt
