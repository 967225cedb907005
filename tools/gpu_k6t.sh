mkdir -p gpurun_out/k6t
for c in C2 C5; do for VT in 33:48 33:64 33:80 33:96 49:96 49:128; do V=${VT%%:*}; T=${VT##*:}; for m in fast matched; do
  HEAT1D_K6_V=$V timeout 300 python bench.py --config $c --T $T --mode $m --no-cpu-baseline --no-e2e --no-other-mode --steps 5 \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$c','V':$V,'T':$T,'mode':'$m','glups':round(d['value'],1),'kernel_ms':d['roofline']['avg_launch_ms'],'kernel':d['roofline']['kernel']}))" >> gpurun_out/k6t/res.jsonl 2>>gpurun_out/k6t/err.log
done; done; done
