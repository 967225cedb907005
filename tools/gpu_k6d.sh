set -x
mkdir -p gpurun_out
for i in 1 2; do for T in 16 32; do timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6d.jsonl 2>> gpurun_out/bench_k6d.err; done; done
timeout 600 python bench.py --config C2 --T 32 --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6d.jsonl 2>> gpurun_out/bench_k6d.err
nvidia-smi -q -d CLOCK,PERFORMANCE > gpurun_out/k6d_smi.txt
