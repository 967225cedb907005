mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ts_pytest.log 2>&1; echo pytest=$?
for T in 12 16 20 24 28 32; do timeout 600 python bench.py --config C4 --T $T --steps 2 --warmup 2 --no-e2e --no-cpu-baseline >> gpurun_out/tsweep_c4.jsonl 2>> gpurun_out/tsweep.err; done
for T in 1 2 4 8 10 12 16 20 24 32; do timeout 600 python bench.py --config C3 --T $T --steps 3 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/tsweep_c3.jsonl 2>> gpurun_out/tsweep.err; done
timeout 600 python bench.py --config C3 --T 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --mode matched >> gpurun_out/tsweep_c3.jsonl 2>> gpurun_out/tsweep.err
