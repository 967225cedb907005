# K6: V selection and period T on the C2 and C5 shapes (variant builds as arguments)
mkdir -p gpurun_out/k6ab
timeout 900 python tools/ab_time.py --variants "$@" --resident True --N 1000000 --nt 1000 --cases 0.5:matched 0.5:fast 0.5:matched:56 0.5:fast:56 0.5:matched:48 0.5:fast:48 0.5:matched:40 0.5:fast:40 > gpurun_out/k6ab/tv_c2.jsonl 2> gpurun_out/k6ab/tv_c2.err; echo c2=$?
timeout 900 python tools/ab_time.py --variants "$@" --resident True --N 1048576 --nt 20000 --cases 0.25:matched 0.25:fast 0.25:matched:56 0.25:fast:56 0.25:matched:48 0.25:fast:48 0.25:matched:40 0.25:fast:40 > gpurun_out/k6ab/tv_c5.jsonl 2> gpurun_out/k6ab/tv_c5.err; echo c5=$?
