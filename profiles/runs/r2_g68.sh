# re-A/B of earlier generator switches on the current kernels (cz-ladder / cnot-ring at 28, 30)
mkdir -p gpurun_out
run() { echo "# $1"; env $1 timeout 500 python profiles/time_jit.py 28 30 2>&1 | grep -v "^{" | python -c "
import sys, json
for l in sys.stdin:
    parts = l.split(' ', 2)
    if len(parts) < 3: continue
    d = json.loads(parts[2])['jit2']
    print(parts[0], parts[1], '%.2f ms' % (d['circuit_s']*1e3))
"; }
for cfg in QSV_DEFAULT=1 QSV_JIT_DIRECT_ANY=1 QSV_JIT_PARTIAL_BARRIERS=0 QSV_JIT_WARP_LOCAL=0 QSV_JIT_NOHOIST=0 QSV_STAGGER_MAX_PHASES=8 QSV_DEFAULT=1; do run $cfg; done > gpurun_out/knobs.txt
cat gpurun_out/knobs.txt
