# Full round check: all GPU tests, smoke, default bench, other configs.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/full_pytest.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/full_bench_c4.json 2> gpurun_out/full_bench_c4.err; echo bench=$?
for c in C1 C2 C3 C5; do timeout 600 python bench.py --config $c > gpurun_out/full_bench_$c.json 2> gpurun_out/full_bench_$c.err; echo $c=$?; done
timeout 600 python bench.py --impl reference > gpurun_out/full_ref_c4.json 2>&1; echo ref=$?
