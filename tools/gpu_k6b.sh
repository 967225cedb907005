set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident" > gpurun_out/pytest_k6b.log 2>&1; echo pytest=$?
for T in 16 32; do timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6b.jsonl 2>> gpurun_out/bench_k6b.err; done
timeout 600 python bench.py --config C2 --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6b.jsonl 2>> gpurun_out/bench_k6b.err
