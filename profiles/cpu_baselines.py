"""CPU baselines of the random-circuit half of the headline metric, timed with
the REFERENCE implementation itself (qsimcore, installed unmodified into
baseline/_ref) on the host cores of the GPU box.  Run once per round on the
box; bench.py attaches the result (profiles/<round>_cpu_baselines.json) to
its random-circuit extras, next to a small live sample it times itself.

Semantics follow the reference harness (bench.py:179-187 ``time_circuit``):
a fresh zero state per repeat, ``perf_counter`` around ``update_state``, the
minimum of the repeats; QSIM_NUM_THREADS = 1 and = nproc (config.py:13-43).

* cfg1: cnot-ring(16) seeds 0..4, full circuits, both thread settings.
* cfg3: VQE ansatz n=24 (284 gates) + TFIM (47 terms), full, nproc threads.
* cfg4: cz-ladder(n, 20, seed 1) at n = 26 / 28 -- the whole circuit is
  infeasible (24.5 s/layer at n=30 measured for the C port), so a sample of
  the first rotation layer and CZ ladder is timed gate by gate and the full
  circuit is extrapolated from the per-kind mean times and the circuit's
  gate counts (labelled "extrapolated").  n=30 is not run on the host: the
  reference's kernels peak at ~63-80 B/amplitude (64-80 GiB at n=30).

    python profiles/cpu_baselines.py [--out profiles/r2_cpu_baselines.json]
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def load_reference():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "qsimcore")):
        sys.path.insert(0, ref)
    import qsimcore
    import qsimcore.bench  # noqa: F401  (generators, time_circuit)
    return qsimcore


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def time_circuit(core, circ, repeats):
    """bench.py:179-187: fresh zero state, wall time of update_state."""
    times = []
    for _ in range(repeats):
        st = core.StateVector(circ.num_qubits)
        t0 = time.perf_counter()
        circ.update_state(st, rng=np.random.default_rng(0))
        times.append(time.perf_counter() - t0)
    return times


def vqe_ansatz(core, n, layers=4, seed=0):
    rng = np.random.default_rng(seed)
    c = core.ParametricCircuit(n)
    for _ in range(layers):
        for i in range(n):
            c.add_parametric_gate(core.ParametricRY(i, rng.uniform(0, 2 * np.pi)))
            c.add_parametric_gate(core.ParametricRZ(i, rng.uniform(0, 2 * np.pi)))
        for i in range(n - 1):
            c.add_gate(core.CNOT(i, i + 1))
    return c


def tfim(core, n):
    obs = core.Observable(n)
    for i in range(n - 1):
        obs.add_operator(-1.0, f"Z {i} Z {i + 1}")
    for i in range(n):
        obs.add_operator(-0.5, f"X {i}")
    return obs


def cfg1(core, threads_list, repeats):
    out = {}
    for th in threads_list:
        core.config.set_num_threads(th)
        per_seed = {}
        for s in range(5):
            c = core.bench.generate_cnot_ring(16, seed=s)
            per_seed[str(s)] = min(time_circuit(core, c, repeats))
        best = min(per_seed.values())
        out[f"threads={th}"] = {"circuit_s_per_seed": per_seed,
                                "sec_per_layer_best": best / 11,
                                "sec_per_layer_mean": float(np.mean(list(per_seed.values()))) / 11}
    return {"workload": "cnot-ring n=16 seeds 0..4 (656 gates, 11 layers), full circuits",
            "semantics": f"time_circuit (bench.py:179-187), min of {repeats} repeats",
            **out}


def cfg3(core, threads):
    core.config.set_num_threads(threads)
    n = 24
    c = vqe_ansatz(core, n)
    obs = tfim(core, n)
    st = core.StateVector(n)
    t0 = time.perf_counter()
    c.update_state(st)
    t1 = time.perf_counter()
    e = obs.get_expectation_value(st)
    t2 = time.perf_counter()
    return {"workload": "VQE ansatz n=24 (284 gates, 4 layers) + TFIM (47 terms), full",
            "threads": threads, "ansatz_s": t1 - t0, "expectation_s": t2 - t1,
            "total_s": t2 - t0, "energy": e}


def cfg4(core, n, threads, sample_qubits):
    """Gate-by-gate times of a sample of cz-ladder(n, 20, 1)'s first rotation
    layer (RZ, RX, RZ on the sampled qubits) and CZ ladder, extrapolated to
    the whole circuit with its per-kind gate counts."""
    core.config.set_num_threads(threads)
    depth = 20
    circ = core.bench.generate_cz_ladder(n, depth, seed=1)
    counts = {}
    for g in circ.gates:
        k = g.name if getattr(g, "name", None) else type(g).__name__
        counts[k] = counts.get(k, 0) + 1
    st = core.StateVector(n)
    first_layer = circ.gates[:3 * n]
    cz_first = [g for g in circ.gates[3 * n:] if (g.name or "") == "CZ"][: max(1, n // 2)]
    pick = [g for g in first_layer if g.targets[0] in sample_qubits]
    pick += [g for g in cz_first if g.controls[0][0] in sample_qubits or g.targets[0] in sample_qubits]
    times = {}
    sampled = []
    for g in pick:
        t0 = time.perf_counter()
        g.apply(st)
        dt = time.perf_counter() - t0
        k = g.name or type(g).__name__
        times.setdefault(k, []).append(dt)
        qs = list(g.targets) + [q for q, _ in g.controls]
        sampled.append(f"{k}@{qs}: {dt:.3f}s")
    mean = {k: float(np.mean(v)) for k, v in times.items()}
    est = sum(counts[k] * mean[k] for k in counts if k in mean)
    missing = [k for k in counts if k not in mean]
    return {"workload": f"cz-ladder n={n} depth={depth} seed=1 ({circ.get_gate_count()} gates)",
            "threads": threads, "kind": "extrapolated",
            "gate_counts": counts, "mean_gate_s": mean, "sampled_gates": sampled,
            "circuit_s_extrapolated": est, "sec_per_layer_extrapolated": est / (depth + 1),
            "unsampled_kinds": missing,
            "how": "per-kind mean of the sampled gates x the circuit's gate count"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(HERE, "r2_cpu_baselines.json"))
    ap.add_argument("--skip-cfg3", action="store_true")
    ap.add_argument("--cfg4-qubits", default="26,28")
    args = ap.parse_args()
    core = load_reference()
    nproc = os.cpu_count() or 1
    rec = {"reference": core.__file__, "cpu_model": cpu_model(), "cores": nproc,
           "numpy": np.__version__, "python": platform.python_version(),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
    try:
        with open("/proc/meminfo") as fh:
            rec["host_mem_gib"] = int(fh.readline().split()[1]) / 2 ** 20
    except OSError:
        pass
    t0 = time.time()
    rec["cfg1"] = cfg1(core, [1, nproc], repeats=3)
    print("cfg1 done", time.time() - t0, flush=True)
    if not args.skip_cfg3:
        rec["cfg3"] = cfg3(core, nproc)
        print("cfg3 done", time.time() - t0, flush=True)
    rec["cfg4"] = {}
    for n in [int(v) for v in args.cfg4_qubits.split(",") if v]:
        sample = sorted({0, n // 3, (2 * n) // 3, n - 1})
        rec["cfg4"][str(n)] = cfg4(core, n, nproc, sample)
        print(f"cfg4 n={n} done", time.time() - t0, flush=True)
    rec["wall_s"] = time.time() - t0
    with open(args.out, "w") as fh:
        json.dump(rec, fh, indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
