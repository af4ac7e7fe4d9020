import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2011_13524_b200 as qs
from paper_2011_13524_b200 import workloads
n = 24
st = qs.QuantumState(n); st.set_Haar_random_state(1)
obs = workloads.tfim_observable(n)
for _ in range(3): obs.get_expectation_value(st)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); obs.get_expectation_value(st); ts.append(time.perf_counter() - t0)
print("wall best %.3f ms median %.3f ms" % (min(ts) * 1e3, sorted(ts)[10] * 1e3))
