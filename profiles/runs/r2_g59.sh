# first (interpreter) run per variant on small states
mkdir -p gpurun_out
for v in 3 4; do echo "# variant $v"; QSV_TILE_VARIANT=$v timeout 300 python profiles/first_run.py 2>&1; done > gpurun_out/first_run.txt
echo "# default" >> gpurun_out/first_run.txt; timeout 300 python profiles/first_run.py >> gpurun_out/first_run.txt 2>&1
cat gpurun_out/first_run.txt
