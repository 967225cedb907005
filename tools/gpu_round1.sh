set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -k "not c3_full and not c4_first and not c5_full" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for T in 4 8 12 16; do timeout 400 python bench.py --config C4 --steps 2 --warmup 1 --T $T --no-cpu-baseline --no-e2e >> gpurun_out/bench_c4.jsonl 2>>gpurun_out/bench_err.log; echo bench$T=$?; done
for T in 8 12; do timeout 300 python bench.py --config C3 --steps 3 --warmup 2 --T $T --no-cpu-baseline --no-e2e >> gpurun_out/bench_c3.jsonl 2>>gpurun_out/bench_err.log; done
timeout 1200 python -m pytest tests -m gpu -x -q -k "c3_full or c4_first or c5_full" > gpurun_out/pytest_gpu_big.log 2>&1; echo pytestbig=$?
