mkdir -p gpurun_out/kx13
HEAT1D_GEOM=49,4,2,2,6 timeout 600 python -m pytest tests -m gpu -q -x -k "c1_bitwise or cross_T or ragged_multi" > gpurun_out/kx13/pytest.log 2>&1; echo pytest=$?
for m in fast matched; do
timeout 900 python tools/sweep.py --N 268435456 --nt 384 --T 64 96 128 --k 0.5 0.4 --mode $m --reps 3 \
  --geoms 49,4,2,2,4 49,4,2,2,6 >> gpurun_out/kx13/sweep.jsonl 2>> gpurun_out/kx13/sweep.err; echo sweep_$m=$?
done
