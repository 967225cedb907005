# Round 2, first GPU pass: exactness-guard parity, C4 bench (both modes), full GPU suite.
mkdir -p gpurun_out/a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_exactness.py -q -x > gpurun_out/a/exact.log 2>&1; echo exact=$?
timeout 600 python bench.py --mode matched --no-cpu-baseline --no-e2e > gpurun_out/a/bench_C4_matched.json 2> gpurun_out/a/bench_C4_matched.err; echo bench=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/a/pytest_gpu.log 2>&1; echo pytest=$?
