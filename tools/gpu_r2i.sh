mkdir -p gpurun_out/i
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -q -x -k "fast or random or solve_host or resident or non_blocking" > gpurun_out/i/fast.log 2>&1; echo fast=$?
timeout 600 python tools/ab_time.py --variants cur2 devrange --cases 0.5:fast 0.4:fast 0.5:matched > gpurun_out/i/ab_k2.jsonl 2>&1; echo abk2=$?
timeout 600 python tools/ab_time.py --variants cur2 devrange --resident True --N 1000000 --nt 1000 --cases 0.5:fast 0.5:matched > gpurun_out/i/ab_c2.jsonl 2>&1; echo abc2=$?
timeout 600 python tools/ab_time.py --variants cur2 devrange --resident True --N 1048576 --nt 20000 --cases 0.25:fast > gpurun_out/i/ab_c5.jsonl 2>&1; echo abc5=$?
for c in C2 C5; do timeout 600 python bench.py --config $c --mode fast --no-cpu-baseline --no-other-mode > gpurun_out/i/bench_fast_$c.json 2> gpurun_out/i/bench_fast_$c.err; echo bench$c=$?; done
