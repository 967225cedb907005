mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "resident or c1_ or tiny or geometries or cross_T or virtual" > gpurun_out/pytest_k6j.log 2>&1; echo pytest=$?
timeout 600 python tools/k6_ab.py --config C5 --nt 4000 > gpurun_out/k6j_ab_c5.jsonl 2>&1
timeout 600 python tools/k6_ab.py --config C2 --nt 1000 > gpurun_out/k6j_ab_c2.jsonl 2>&1
timeout 900 python tools/sweep.py --nt 1200 --geoms 17,8,3,2,0 17,8,3,2,1 17,8,3,2,2 33,4,3,2,2 17,8,2,3,2 --T 8 12 16 --k 0.4 0.5 > gpurun_out/sweep6.jsonl 2> gpurun_out/sweep6.err
