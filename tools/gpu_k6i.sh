mkdir -p gpurun_out
export HEAT1D_K6_SPW=1 HEAT1D_K6_EARLY=0 HEAT1D_K6_RELAXED=1
CMD="python bench.py --config C5 --nt 640 --T 32 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/k6i_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k6 -s 1 -c 1 -o gpurun_out/k6i $CMD > gpurun_out/ncu_k6i.log 2>&1; echo ncu=$?
