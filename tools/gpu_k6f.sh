set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or c1_ or tiny" > gpurun_out/pytest_k6f.log 2>&1; echo pytest=$?
for spw in 1 2; do for T in 16 32; do HEAT1D_K6_SPW=$spw timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline --steps 2 --warmup 2 >> gpurun_out/bench_k6f.jsonl 2>> gpurun_out/bench_k6f.err; done; done
for spw in 1 2; do HEAT1D_K6_SPW=$spw timeout 600 python bench.py --config C2 --T 32 --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6f.jsonl 2>> gpurun_out/bench_k6f.err; done
