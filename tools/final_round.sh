# Round-end measurement pass (run under gpurun): profile_round.sh (bench line,
# launch list, ncu captures) plus the path-only, PPO and DAPO bench lines.
# Usage: bash tools/final_round.sh <tag>
T=${1:-v9}
bash tools/profile_round.sh $T > gpurun_out/profile_$T.log 2>&1
timeout 600 python bench.py --verify path > gpurun_out/bench_grpo_path_$T.log 2>&1
timeout 600 python bench.py --config ppo > gpurun_out/bench_ppo_$T.log 2>&1
timeout 900 python bench.py --config dapo > gpurun_out/bench_dapo_$T.log 2>&1
ls gpurun_out
