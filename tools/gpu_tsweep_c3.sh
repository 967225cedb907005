# north_star: "The choice of T is justified by ncu-measured HBM GB/s and the FP64 pipe utilisation":
# C3 bench lines per T and mode, plus one ncu metrics capture of a K2 launch per (T, mode).
mkdir -p gpurun_out/ts
timeout 900 python -m pytest tests -m gpu -q -x -k "c4_full_nt" > gpurun_out/ts/pytest_c4full.log 2>&1; echo pytest=$?
for m in fast matched; do for T in 1 2 4 8 16 32 64 128; do
  timeout 600 python bench.py --config C3 --T $T --mode $m --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-other-mode >> gpurun_out/ts/bench_c3.jsonl 2>> gpurun_out/ts/err.log
done; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second
for m in fast matched; do for T in 1 2 4 8 16 32 64 128; do
  ncu --metrics $M --clock-control none -k regex:k2p -s 2 -c 1 --csv python bench.py --config C3 --T $T --mode $m --nt $((4*T)) --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode > gpurun_out/ts/ncu_${m}_T$T.csv 2>> gpurun_out/ts/err.log
done; done
echo done
