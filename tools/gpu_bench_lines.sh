# smoke, the default bench line (C4, matched headline), the multi-slab overlap trace, other configs
mkdir -p gpurun_out/c
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/c/bench_C4.json 2> gpurun_out/c/bench_C4.err; echo benchC4=$?
timeout 900 python tools/overlap_trace.py --config C4 --nt 1000 --slabs 8 --out gpurun_out/c/overlap_c4.json > gpurun_out/c/overlap.log 2>&1; echo overlap=$?
for c in C3 C5 C2 C1; do timeout 600 python bench.py --config $c > gpurun_out/c/bench_$c.json 2> gpurun_out/c/bench_$c.err; echo bench$c=$?; done
