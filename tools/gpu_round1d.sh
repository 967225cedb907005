set -x
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --geoms 17,8,3,2,0 17,8,2,3,0 17,6,2,4,0 17,6,3,3,0 17,12,2,2,0 17,16,2,1,0 15,8,2,3,0 15,8,3,2,0 33,4,3,2,0 25,4,3,2,0 17,4,3,4,0 --T 8 12 16 --k 0.4 0.5 > gpurun_out/sweep3.jsonl 2> gpurun_out/sweep3.err; echo sweep=$?
CMD="python tools/sweep.py --N 67108864 --nt 24 --T 12 --k 0.5 --reps 1 --geoms 17,8,3,2,1"
$CMD > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2w_pass -s 2 -c 1 -o gpurun_out/k2w_T12 $CMD > gpurun_out/ncu_run2.log 2>&1; echo ncu=$?
