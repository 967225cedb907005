set -x
mkdir -p gpurun_out
CMD="python bench.py --config C5 --nt 640 --T 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/k6_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k6 -s 1 -c 1 -o gpurun_out/k6_c5_spw2 $CMD > gpurun_out/ncu_k6_2.log 2>&1; echo ncu=$?
