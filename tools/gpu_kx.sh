# kind 4 geometries and T up to 128: tests and sweep
mkdir -p gpurun_out/kx3
timeout 900 python -m pytest tests -m gpu -q -x -k "interwarp or geometries or c1_bitwise or cross_T" > gpurun_out/kx3/pytest.log 2>&1; echo pytest=$?
for m in fast matched; do
timeout 900 python tools/sweep.py --N 268435456 --nt 384 --T 32 48 64 96 128 --k 0.5 0.4 --mode $m --reps 2 \
  --geoms 33,4,3,2,2 49,4,2,2,4 41,4,2,2,4 53,4,2,2,4 49,8,2,1,4 65,4,2,1,4 >> gpurun_out/kx3/sweep.jsonl 2>> gpurun_out/kx3/sweep.err; echo sweep_$m=$?
done
