# Bench lines with the fast headline + matched other mode; GPU suite.
mkdir -p gpurun_out/f3
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f3/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/f3/bench_C4.json 2> gpurun_out/f3/bench_C4.err; echo C4=$?
for c in C3 C5 C2 C1; do timeout 600 python bench.py --config $c > gpurun_out/f3/bench_$c.json 2> gpurun_out/f3/bench_$c.err; echo $c=$?; done
