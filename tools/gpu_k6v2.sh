mkdir -p gpurun_out/k6v2
for c in C2 C5; do for VT in 29:64 33:64 37:64 41:64 37:80 41:96; do V=${VT%%:*}; T=${VT##*:}; for m in fast matched; do
  HEAT1D_K6_V=$V timeout 300 python bench.py --config $c --T $T --mode $m --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','V':$V,'T':$T,'mode':'$m','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms']}))" >> gpurun_out/k6v2/res.jsonl 2>>gpurun_out/k6v2/err.log
done; done; done
