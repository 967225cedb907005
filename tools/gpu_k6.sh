set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or ragged or c1_ or cross_T or tiny or c2_" > gpurun_out/pytest_k6.log 2>&1; echo pytest=$?
for c in C1 C2 C5; do timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6.jsonl 2>> gpurun_out/bench_k6.err; echo $c=$?; done
for T in 8 12 24 32; do timeout 600 python bench.py --config C5 --T $T --no-e2e --no-cpu-baseline >> gpurun_out/bench_k6.jsonl 2>> gpurun_out/bench_k6.err; done
