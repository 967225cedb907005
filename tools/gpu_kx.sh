mkdir -p gpurun_out/kx16
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/kx16/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "c3_ or c4_ or geometries or interwarp or random or solve_host" > gpurun_out/kx16/pytest.log 2>&1; echo pytest=$?
for c in C4 C3; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['other_mode']['value']), round(d['other_mode']['roofline']['frac'],3))"; done
