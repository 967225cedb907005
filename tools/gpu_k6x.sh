# K6: period T=32 vs 64 (V=17 vs 33) and the three acquire patterns, on C5 and C2
mkdir -p gpurun_out/k6x
timeout 900 python -m pytest tests -m gpu -q -x -k "resident" > gpurun_out/k6x/pytest.log 2>&1; echo pytest=$?
for c in C5 C2; do for T in 32 64; do for s in 0 1 2; do for m in fast matched; do
  HEAT1D_K6_SYNC=$s timeout 300 python bench.py --config $c --T $T --mode $m --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','T':$T,'sync':$s,'mode':'$m','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms'],'step_ms':d['ms_per_step']}))" >> gpurun_out/k6x/res.jsonl 2>>gpurun_out/k6x/err.log
done; done; done; done
echo done
