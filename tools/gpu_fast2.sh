# T > 32 sweep for all arithmetic variants + full GPU suite.
mkdir -p gpurun_out/f2
for m in fast matched; do
timeout 900 python tools/sweep.py --N 268435456 --nt 384 --T 24 32 40 48 64 --k 0.5 0.4 --mode $m --reps 2 \
  --geoms 33,4,3,2,2 49,4,3,2,2 25,4,3,2,2 33,8,3,1,2 >> gpurun_out/f2/sweep.jsonl 2>> gpurun_out/f2/sweep.err; echo sweep_$m=$?
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f2/pytest_gpu.log 2>&1; echo pytest=$?
