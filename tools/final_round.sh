bash tools/profile_round.sh v8 > gpurun_out/profile_v8.log 2>&1
timeout 600 python bench.py --verify path > gpurun_out/bench_grpo_path_v8.log 2>&1
timeout 600 python bench.py --config ppo > gpurun_out/bench_ppo_v8.log 2>&1
timeout 900 python bench.py --config dapo > gpurun_out/bench_dapo_v8b.log 2>&1
ls gpurun_out
