bash tools/profile_r02.sh v6
SRT_STREAM_HINT=1 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/v6/bench_grpo_streamhint1.log 2>&1
