mkdir -p gpurun_out/j
HEAT1D_DEBUG=1 timeout 600 python tools/ab_time.py --variants k6base k6v49 --resident True --N 1000000 --nt 1000 --cases 0.5:matched:64 0.5:fast:64 > gpurun_out/j/ab_c2.jsonl 2> gpurun_out/j/ab_c2.err; echo abc2=$?
HEAT1D_DEBUG=1 timeout 600 python tools/ab_time.py --variants k6base k6v49 --resident True --N 1048576 --nt 20000 --cases 0.25:matched:64 0.25:fast:64 > gpurun_out/j/ab_c5.jsonl 2> gpurun_out/j/ab_c5.err; echo abc5=$?
