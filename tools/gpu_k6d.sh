mkdir -p gpurun_out/k6d
for args in "--T 64" "" ; do for env in "HEAT1D_K6_V=33" "X=1"; do
  env $env timeout 300 python bench.py --config C5 --mode matched $args --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'args':'$args','env':'$env','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms'],'kernel':d['roofline']['kernel'],'T':d['config']['T'],'ops':d['config']['dp_ops']}))" >> gpurun_out/k6d/res.jsonl 2>>gpurun_out/k6d/err.log
done; done
