mkdir -p gpurun_out/kx10
for m in fast matched; do
timeout 900 python tools/sweep.py --N 268435456 --nt 384 --T 64 96 --k 0.5 0.4 --mode $m --reps 3 \
  --geoms 49,4,2,2,4 >> gpurun_out/kx10/sweep.jsonl 2>> gpurun_out/kx10/sweep.err; echo sweep_$m=$?
done
