set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "geometries or ragged or c1_ or cross_T or virtual" > gpurun_out/pytest_g.log 2>&1; echo pytest=$?
timeout 900 python tools/sweep.py --nt 1200 --geoms 17,8,3,2,0 17,8,3,2,2 17,8,4,1,2 17,8,2,3,2 17,4,4,3,2 33,4,3,2,0 33,4,3,2,2 25,4,3,2,2 15,8,3,2,2 17,16,2,1,2 --T 8 12 16 --k 0.4 0.5 > gpurun_out/sweep5.jsonl 2> gpurun_out/sweep5.err; echo sweep=$?
CMD="python tools/sweep.py --N 67108864 --nt 24 --T 12 --k 0.4 0.5 --reps 1 --geoms 17,8,3,2,2 17,8,4,1,2"
$CMD > gpurun_out/ncu_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2 -s 2 -c 8 -o gpurun_out/k2p_T12 $CMD > gpurun_out/ncu_run5.log 2>&1; echo ncu=$?
