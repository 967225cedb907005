mkdir -p gpurun_out
timeout 600 python bench.py --config C5 --T 32 --no-e2e --no-cpu-baseline > gpurun_out/k6h_bench.json 2>&1
timeout 600 python tools/k6_ab.py --config C5 --nt 20000 --T 32 --reps 2 > gpurun_out/k6h_ab20000.jsonl 2>&1
timeout 600 python tools/k6_ab.py --config C5 --nt 2000 --T 32 --reps 2 > gpurun_out/k6h_ab2000.jsonl 2>&1
timeout 600 python tools/k6_ab.py --config C5 --nt 200 --T 32 --reps 2 > gpurun_out/k6h_ab200.jsonl 2>&1
