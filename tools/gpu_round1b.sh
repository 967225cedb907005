set -x
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --geoms 17,8,3,2 17,8,2,2 17,8,4,1 17,4,3,4 17,4,4,3 21,8,3,1 21,4,3,2 25,4,3,2 25,8,2,1 33,4,3,2 33,8,2,1 9,8,4,2 9,4,4,4 --T 8 12 16 --k 0.4 0.5 > gpurun_out/sweep1.jsonl 2> gpurun_out/sweep1.err; echo sweep=$?
CMD="python tools/sweep.py --N 67108864 --nt 24 --T 12 --k 0.4 0.5 --reps 1"
$CMD > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 2 -c 2 -o gpurun_out/k2_T12 $CMD > gpurun_out/ncu_run.log 2>&1; echo ncu=$?
