# A/B of K6 variants (tools/ab_build.py names as arguments) on the C2 and C5 shapes
mkdir -p gpurun_out/k6ab
timeout 600 python tools/ab_time.py --variants "$@" --resident True --N 1000000 --nt 1000 --cases 0.5:matched 0.5:fast > gpurun_out/k6ab/c2.jsonl 2> gpurun_out/k6ab/c2.err; echo c2=$?
timeout 600 python tools/ab_time.py --variants "$@" --resident True --N 1048576 --nt 20000 --cases 0.25:matched 0.25:fast > gpurun_out/k6ab/c5.jsonl 2> gpurun_out/k6ab/c5.err; echo c5=$?
