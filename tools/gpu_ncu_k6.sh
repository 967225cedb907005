# ncu --set full: K6 on C2 (matched), after the same command ran clean
mkdir -p gpurun_out/ncu6
CMD="python bench.py --config C2 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode --no-parity"
$CMD > gpurun_out/ncu6/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k6_resident -c 1 -o gpurun_out/ncu6/k6_c2_matched $CMD > gpurun_out/ncu6/ncu_c2.log 2>&1; echo c2=$?
