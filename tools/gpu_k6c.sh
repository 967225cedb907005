set -x
mkdir -p gpurun_out
for d in 0 1; do for T in 16 32; do HEAT1D_K6_DEBUG=$d timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline --steps 2 --warmup 1 >> gpurun_out/bench_k6c.jsonl 2>> gpurun_out/bench_k6c.err; done; done
