mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or c1_ or tiny" > gpurun_out/pytest_k6g.log 2>&1; echo pytest=$?
timeout 600 python tools/k6_ab.py --config C5 > gpurun_out/k6_ab_c5.jsonl 2>&1; echo ab=$?
timeout 600 python tools/k6_ab.py --config C2 --nt 1000 > gpurun_out/k6_ab_c2.jsonl 2>&1; echo ab2=$?
