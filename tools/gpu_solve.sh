mkdir -p gpurun_out/sv
timeout 900 python -m pytest tests -m gpu -q -x -k "solve_host" > gpurun_out/sv/pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py --no-cpu-baseline --no-other-mode > gpurun_out/sv/bench_C4.json 2> gpurun_out/sv/bench_C4.err; echo C4=$?
timeout 900 python bench.py --config C3 --no-cpu-baseline --no-other-mode > gpurun_out/sv/bench_C3.json 2> gpurun_out/sv/bench_C3.err; echo C3=$?
