mkdir -p gpurun_out/k6y
timeout 900 python -m pytest tests -m gpu -q -x -k "resident or bench" > gpurun_out/k6y/pytest.log 2>&1; echo pytest=$?
for c in C5 C2; do for T in 64 96 128; do for m in fast matched; do
  timeout 300 python bench.py --config $c --T $T --mode $m --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','T':$T,'mode':'$m','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms'],'step_ms':d['ms_per_step'],'kernel':d['roofline']['kernel']}))" >> gpurun_out/k6y/res.jsonl 2>>gpurun_out/k6y/err.log
done; done; done
timeout 600 python bench.py > gpurun_out/k6y/bench_C4.json 2>/dev/null; echo C4=$?
