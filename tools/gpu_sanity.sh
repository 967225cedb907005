# Quick sanity on a fresh box: smoke, GPU parity tests, default bench line.
mkdir -p gpurun_out/s
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s/bench_C4.json 2> gpurun_out/s/bench_C4.err; echo bench=$?
