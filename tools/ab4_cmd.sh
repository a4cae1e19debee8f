# rank-based full-scan hub refresh (fused step fallback + k_hub_refresh): parity, then A/B
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ab4_pytest.log 2>&1; tail -2 gpurun_out/ab4_pytest.log
bash tools/probe_ab.sh ab4 base3 grpo ppo dapo
