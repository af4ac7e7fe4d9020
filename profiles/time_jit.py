"""Device time of benchmark circuits with the tile-pass interpreter (jit=0)
and with generated pass kernels (jit=2), plus the NVRTC compile / cache
cost.  python profiles/time_jit.py [n ...]"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/profiles/", 1)[0])
import paper_2011_13524_b200 as qs  # noqa: E402
from paper_2011_13524_b200 import workloads  # noqa: E402
from paper_2011_13524_b200._lib import jit_stats  # noqa: E402


def dev_time(circ, st, reps=3):
    s = torch.cuda.current_stream()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        circ.update_quantum_state(st)
        b.record(s)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


def main():
    ns = [int(v) for v in sys.argv[1:]] or [30]
    out = {}
    for n in ns:
        fams = {"cz-ladder": lambda: workloads.generate_cz_ladder(n, 20, seed=1),
                "cnot-ring": lambda: workloads.generate_cnot_ring(n, seed=1)}
        if n <= 26:
            fams["vqe"] = lambda: workloads.vqe_ansatz(n)
        for name, make in fams.items():
            rec = {}
            for jit in (0, 2):
                circ = make()
                t0 = time.perf_counter()
                circ.set_plan_options(jit=jit)
                stats = circ.program_stats()
                plan_s = time.perf_counter() - t0
                st = qs.QuantumState(n)
                st.set_stream(torch.cuda.current_stream().cuda_stream)
                st.set_random_state_device(5)
                circ.update_quantum_state(st)
                circ.update_quantum_state(st)
                torch.cuda.synchronize()
                t = dev_time(circ, st)
                rec[f"jit{jit}"] = {"circuit_s": t, "sec_per_layer": t / (21 if name == "cz-ladder" else 11),
                                    "plan_and_compile_s": plan_s, "passes": stats["num_tile_passes"],
                                    "jit_passes": circ.program_stats()["num_jit_passes"],
                                    "fp64_tflops": stats["fp64_flops"] / t / 1e12}
                del st
            out[f"{name}/{n}"] = rec
            print(name, n, json.dumps(rec), flush=True)
    out["jit_stats"] = jit_stats()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
