# Fast-mode (scaled state) variants: parity tests, then bench lines for C4 / C3 / C5.
mkdir -p gpurun_out/f1
timeout 900 python -m pytest tests -m gpu -q -x -k "fast" > gpurun_out/f1/pytest_fast.log 2>&1; echo pytest=$?
for c in C4 C3 C5 C2; do timeout 600 python bench.py --config $c --mode fast --no-cpu-baseline --no-e2e > gpurun_out/f1/bench_$c.json 2> gpurun_out/f1/bench_$c.err; echo $c=$?; done
timeout 600 python tools/sweep.py --N 268435456 --nt 256 --T 8 16 24 32 --k 0.5 0.4 --mode fast --reps 2 > gpurun_out/f1/sweep.jsonl 2>&1; echo sweep=$?
