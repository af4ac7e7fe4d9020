# phase cap per pass revisited with the current kernels (cz-ladder / cnot-ring at 28, 30)
mkdir -p gpurun_out
for cap in 0 10 12 14; do echo "# cap $cap"; if [ $cap = 0 ]; then timeout 500 python profiles/time_jit.py 28 30; else QSV_MAX_PASS_PHASES=$cap timeout 500 python profiles/time_jit.py 28 30; fi 2>&1 | grep -v "^{" | python -c "
import sys, json
for l in sys.stdin:
    parts = l.split(' ', 2)
    if len(parts) < 3: continue
    d = json.loads(parts[2])['jit2']
    print(parts[0], parts[1], '%.2f ms' % (d['circuit_s']*1e3), d['passes'], 'passes')
"; done > gpurun_out/cap.txt
cat gpurun_out/cap.txt
