# ncu evidence for the fast-mode headline (C4, k2p_pass<OPS=1>, T=64) and matched (OPS=3, T=32).
mkdir -p gpurun_out/n1
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode"
$CMD > gpurun_out/n1/plain.log 2>&1; echo plain=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/n1/launches_C4.csv $CMD > gpurun_out/n1/ncu_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/n1/k2p_C4_fast $CMD > gpurun_out/n1/ncu_full.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k2p -s 20 -c 1 -o gpurun_out/n1/k2p_C4_matched $CMD --mode matched > gpurun_out/n1/ncu_full_m.log 2>&1; echo ncu3=$?
