# Round-2 re-entry pass (run under gpurun): GPU tests, default bench line,
# lmhead bench line, PPO/DAPO lines, sanitizer logs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; tail -3 gpurun_out/pt_all.log
timeout 400 python bench.py > gpurun_out/bench_grpo.log 2>&1; tail -1 gpurun_out/bench_grpo.log | cut -c1-400
timeout 400 python bench.py --verify lmhead --no-cpu-baseline > gpurun_out/bench_lmhead.log 2>&1; tail -1 gpurun_out/bench_lmhead.log | cut -c1-400
timeout 400 python bench.py --config ppo --no-cpu-baseline > gpurun_out/bench_ppo.log 2>&1
timeout 600 python bench.py --config dapo --no-cpu-baseline > gpurun_out/bench_dapo.log 2>&1
timeout 400 python bench.py --sharded --no-cpu-baseline > gpurun_out/bench_sharded.log 2>&1
ls gpurun_out
