# A/B timing of variant builds (tools/ab_build.py -> tools/ab_time.py); args: variant names
mkdir -p gpurun_out/ab
timeout 1200 python tools/ab_time.py --variants "$@" --cases ${AB_CASES:-0.5:matched 0.4:matched 0.5:fast} > gpurun_out/ab/ab.jsonl 2> gpurun_out/ab/ab.err; echo ab=$?
