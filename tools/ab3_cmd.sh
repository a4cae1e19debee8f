# rank-based incremental hub refresh: parity (fused step vs separate, full-size vs the oracle), then A/B
timeout 1200 python -m pytest tests/test_gpu_bench.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ab3_pytest.log 2>&1; tail -2 gpurun_out/ab3_pytest.log
SRT_STEP_PROF=1 timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 6 --warmup 3 2>&1 | grep "tree step" | tail -2 > gpurun_out/ab3_stepprof.txt
bash tools/probe_ab.sh ab3 base2 grpo ppo dapo
