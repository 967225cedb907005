# K6 configs: the GPU suite, then the bench lines of C1, C2, C5 (on-chip rings)
mkdir -p gpurun_out/k6l
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/k6l/pytest.txt 2>&1; echo pytest=$?
for c in C5 C2 C1; do timeout 600 python bench.py --config $c > gpurun_out/k6l/bench_$c.json 2> gpurun_out/k6l/bench_$c.err; echo bench$c=$?; done
