set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "geometries or ragged or c1_ or cross_T or virtual" > gpurun_out/pytest_f.log 2>&1; echo pytest=$?
CMD="python tools/sweep.py --N 67108864 --nt 24 --T 12 --k 0.4 0.5 --reps 1 --geoms 17,8,3,2,0 17,8,3,2,1 33,4,3,2,0"
$CMD > gpurun_out/ncu_plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2 -s 2 -c 12 -o gpurun_out/k2_v3_T12 $CMD > gpurun_out/ncu_run4.log 2>&1; echo ncu=$?
