mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "geometries or c1_ or resident" > gpurun_out/vs_pytest.log 2>&1; echo pytest=$?
timeout 1200 python tools/sweep.py --nt 1920 --geoms 33,4,3,2,2 41,4,3,2,2 49,4,3,2,2 49,2,3,3,2 65,2,3,2,2 65,2,4,1,2 33,6,3,1,2 33,8,4,1,2 33,4,3,2,0 --T 16 24 32 --k 0.4 0.5 > gpurun_out/sweep7.jsonl 2> gpurun_out/sweep7.err
