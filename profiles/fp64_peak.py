"""Run profiles/micro/fp64_peak.cu on the GPU with nvidia-smi clock sampling
and write profiles/fp64_peak.json (FP64 DFMA burst / sustained peaks and the
DMMA .f64 tensor-core rates, with the SM clocks and throttle reasons seen
while they ran).  bench.py grades the tile kernel against the sustained DFMA
figure.

    python profiles/fp64_peak.py
"""

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from bench import ClockSampler  # noqa: E402


def main():
    src = os.path.join(HERE, "micro", "fp64_peak.cu")
    exe = os.path.join(HERE, "micro", "fp64_peak")
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", src, "-o", exe],
                   check=True)
    with ClockSampler(0) as clk:
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    rec = json.loads(out.strip().splitlines()[-1])
    rec["clocks"] = clk.summary()
    gpu = subprocess.run(["nvidia-smi", "--query-gpu=name", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    rec["gpu"] = gpu
    with open(os.path.join(HERE, "fp64_peak.json"), "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
