# comm tests; small-state pass durations (ncu launch list) vs the device time of the whole circuit
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_comm.py -q 2>&1 | tail -5 > gpurun_out/pytest_comm.txt
for fam in cnot-ring cz-ladder; do
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none -k regex:k_pass --csv python profiles/prof_jit.py $fam 16 2 > gpurun_out/small16_$fam.csv 2>&1
done
cat gpurun_out/pytest_comm.txt
