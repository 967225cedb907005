set -x
mkdir -p gpurun_out
CMD="python bench.py --config C5 --nt 640 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/k6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k6 -s 1 -c 1 -o gpurun_out/k6_c5 $CMD > gpurun_out/ncu_k6.log 2>&1; echo ncu=$?
