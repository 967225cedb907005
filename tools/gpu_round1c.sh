set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "geometries or ragged or c1_ or tiny or virtual or cross_T" > gpurun_out/pytest_c.log 2>&1; echo pytest=$?
timeout 900 python tools/sweep.py --geoms 17,8,3,2,0 17,8,3,2,1 17,8,2,2,1 17,4,3,4,1 17,4,2,4,1 21,8,3,1,1 25,4,3,2,1 25,4,2,3,1 25,8,2,1,1 33,4,2,2,1 33,8,2,1,1 9,8,4,2,1 --T 8 12 16 --k 0.4 0.5 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err; echo sweep=$?
