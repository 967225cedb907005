# DRAM bytes of one launch of the dominant kernel per (config, mode), for the bench lines' traffic
mkdir -p gpurun_out/tr
for c in C3 C2 C5; do for m in fast matched; do
  K=k2p; [ $c != C3 ] && K=k6
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:$K -c 1 --csv python bench.py --config $c --mode $m --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-other-mode > gpurun_out/tr/${c}_$m.csv 2> gpurun_out/tr/${c}_$m.err; echo $c$m=$?
done; done
