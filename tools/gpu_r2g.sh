mkdir -p gpurun_out/g
timeout 600 python tools/ab_time.py --variants cur --resident True --N 1000000 --nt 1000 --cases 0.5:matched:32 0.5:matched:64 0.5:matched:96 0.5:matched:128 0.5:fast:64 0.5:fast:96 0.5:fast:128 > gpurun_out/g/ab_c2.jsonl 2> gpurun_out/g/ab_c2.err; echo abc2=$?
timeout 600 python tools/ab_time.py --variants cur --resident True --N 1048576 --nt 20000 --cases 0.25:matched:64 0.25:matched:96 0.25:matched:128 0.25:fast:64 0.25:fast:96 0.25:fast:128 > gpurun_out/g/ab_c5.jsonl 2> gpurun_out/g/ab_c5.err; echo abc5=$?
