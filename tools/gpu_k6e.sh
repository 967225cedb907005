set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or c1_ or cross_T or tiny or c2_ or ragged" > gpurun_out/pytest_k6e.log 2>&1; echo pytest=$?
for T in 16 24 32; do timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6e.jsonl 2>> gpurun_out/bench_k6e.err; done
for T in 16 32; do timeout 600 python bench.py --config C2 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6e.jsonl 2>> gpurun_out/bench_k6e.err; done
