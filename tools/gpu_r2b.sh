# exactness + full GPU suite on the folded-guard build; K6 guard cost A/B (C5, C2 shapes)
mkdir -p gpurun_out/b
timeout 900 python -m pytest tests/test_gpu_exactness.py -q -x > gpurun_out/b/exact.log 2>&1; echo exact=$?
timeout 600 python tools/ab_time.py --variants noguard2 fold --resident True --N 1048576 --nt 20000 --cases 0.25:matched 0.25:fast > gpurun_out/b/ab_k6_c5.jsonl 2>&1; echo abk6=$?
timeout 600 python tools/ab_time.py --variants noguard2 fold --resident True --N 1000000 --nt 1000 --cases 0.5:matched 0.5:fast > gpurun_out/b/ab_k6_c2.jsonl 2>&1; echo abk6b=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/b/pytest_gpu.log 2>&1; echo pytest=$?
