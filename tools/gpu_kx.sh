mkdir -p gpurun_out/kx12
timeout 600 python -m pytest tests -m gpu -q -x -k "interwarp" > gpurun_out/kx12/pytest.log 2>&1; echo pytest=$?
for m in fast matched; do
timeout 900 python tools/sweep.py --N 268435456 --nt 384 --T 64 96 --k 0.5 0.4 --mode $m --reps 3 \
  --geoms 49,4,2,2,4 >> gpurun_out/kx12/sweep.jsonl 2>> gpurun_out/kx12/sweep.err; echo sweep_$m=$?
done
