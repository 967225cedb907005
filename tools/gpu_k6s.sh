mkdir -p gpurun_out/k6s4
HEAT1D_K6_SYNC=3 timeout 900 python -m pytest tests -m gpu -q -x -k "resident" > gpurun_out/k6s4/pytest3.log 2>&1; echo pytest3=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "sync_variants" > gpurun_out/k6s4/pytest.log 2>&1; echo pytest=$?
for c in C2 C5; do for sy in 0 3; do for m in fast matched; do
  HEAT1D_K6_SYNC=$sy timeout 300 python bench.py --config $c --mode $m --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','sync':$sy,'mode':'$m','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms']}))" >> gpurun_out/k6s4/res.jsonl 2>>gpurun_out/k6s4/err.log
done; done; done
