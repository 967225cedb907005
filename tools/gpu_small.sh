set -x
mkdir -p gpurun_out
for c in C1 C2 C5; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline >> gpurun_out/bench_small_rings.jsonl 2>> gpurun_out/bench_small_rings.err; echo $c=$?; done
for T in 8 16 32; do timeout 600 python bench.py --config C2 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_small_rings.jsonl 2>> gpurun_out/bench_small_rings.err; done
