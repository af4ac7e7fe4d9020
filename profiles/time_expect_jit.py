"""Expectation value of the TFIM observable (cfg3 Hamiltonian) with the
generated pass kernels (default) or the generic k_expect_tile
(QSV_EXPECT_JIT=0): wall and device time per evaluation, HBM fraction per
pass.  python profiles/time_expect_jit.py [n ...]"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads, _lib  # noqa: E402

PEAK = 6536.4e9  # MEASURED_PEAKS.json copy bandwidth, B/s


def main():
    out = {"mode": os.environ.get("QSV_EXPECT_JIT", "1")}
    for n in [int(v) for v in sys.argv[1:]] or [24, 28]:
        obs = workloads.tfim_observable(n)
        st = qs.QuantumState(n)
        s = torch.cuda.current_stream()
        st.set_stream(s.cuda_stream)
        st.set_random_state_device(3)
        t0 = time.perf_counter()
        v0 = obs.get_expectation_value(st)
        first = time.perf_counter() - t0
        t0 = time.perf_counter()
        v1 = obs.get_expectation_value(st)
        second = time.perf_counter() - t0
        p0 = _lib.expect_path_stats()
        walls, devs = [], []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a.record(s)
            v = obs.get_expectation_value(st)
            b.record(s)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
            devs.append(a.elapsed_time(b) / 1e3)
        p1 = _lib.expect_path_stats()
        passes = (p1["jit_passes"] - p0["jit_passes"] + p1["generic_passes"]
                  - p0["generic_passes"]) / 10
        dev = min(devs)
        floor = passes * 16 * 2 ** n / PEAK
        rec = {"terms": obs.get_term_count(), "value": v, "first_eval_s": first,
               "second_eval_s": second, "wall_s": min(walls), "device_s": dev,
               "passes": passes, "hbm_floor_s": floor, "hbm_frac": floor / dev,
               "agree_first_second": abs(v0 - v1), "path": p1}
        out[str(n)] = rec
        print(n, json.dumps(rec), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
