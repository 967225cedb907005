# DRAM bytes of one launch of the dominant kernel per (config, mode), for the bench lines' traffic
# (turn each report into profiles/ncu_traffic.json entries with tools/ncu_summary.py traffic)
mkdir -p gpurun_out/tr
for c in C3 C2 C5; do for m in fast matched; do
  K=k2f_pass; [ $c != C3 ] && K=k6_resident
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:$K -c 1 \
      -o gpurun_out/tr/${c}_$m python bench.py --config $c --mode $m --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
      --no-other-mode --no-parity > gpurun_out/tr/${c}_$m.log 2>&1; echo $c$m=$?
done; done
