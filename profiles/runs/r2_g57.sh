# n = 17..22: r3 (L 10/11) vs r4 (auto / 11 / 12) under generated kernels
mkdir -p gpurun_out
echo "# r4" > gpurun_out/mid_n.txt
QSV_TILE_VARIANT=4 LS=-1,11,12 NS=17,18,19,20,21,22 timeout 400 python profiles/time_small_n.py >> gpurun_out/mid_n.txt 2>&1
echo "# r3" >> gpurun_out/mid_n.txt
QSV_TILE_VARIANT=3 LS=10,11 NS=17,18,19,20,21,22 timeout 400 python profiles/time_small_n.py >> gpurun_out/mid_n.txt 2>&1
echo "# default" >> gpurun_out/mid_n.txt
LS=-1 NS=17,18,19,20,21,22 timeout 400 python profiles/time_small_n.py >> gpurun_out/mid_n.txt 2>&1
cat gpurun_out/mid_n.txt
