mkdir -p gpurun_out/kx14
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/kx14/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "c3_ or c4_first or geometries or interwarp or random" > gpurun_out/kx14/pytest.log 2>&1; echo pytest=$?
for c in C3 C4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), d['roofline']['kernel'], round(d['other_mode']['value']), d['other_mode']['roofline']['kernel'])"; done
