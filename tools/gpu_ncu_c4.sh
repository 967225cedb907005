# ncu evidence for the headline (C4, matched): the launch list of a short bench command, and one
# --set full capture of the dominant kernel (K2 feed tiles, 3-op guarded, T = 128), each after the same command ran clean
mkdir -p gpurun_out/ncu
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-other-mode --no-parity"
$CMD > gpurun_out/ncu/plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu/launches_c4.csv $CMD > gpurun_out/ncu/ncu1.log 2>&1; echo launches=$?
CMD2="python bench.py --steps 1 --warmup 0 --nt 256 --no-e2e --no-cpu-baseline --no-other-mode --no-parity"
$CMD2 > gpurun_out/ncu/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2f_pass -s 1 -c 1 -o gpurun_out/ncu/k2f_c4_matched $CMD2 > gpurun_out/ncu/ncu2.log 2>&1; echo full=$?
# the fast 1-op pass (T = 128) too
CMD3="python bench.py --mode fast --steps 1 --warmup 0 --nt 256 --no-e2e --no-cpu-baseline --no-other-mode --no-parity"
$CMD3 > gpurun_out/ncu/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2f_pass -s 1 -c 1 -o gpurun_out/ncu/k2f_c4_fast $CMD3 > gpurun_out/ncu/ncu3.log 2>&1; echo fast=$?
