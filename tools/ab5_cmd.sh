# rank-sorted merge of a round's children in the draft: parity, then A/B
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ab5_pytest.log 2>&1; tail -2 gpurun_out/ab5_pytest.log
bash tools/probe_ab.sh ab5 base4 grpo ppo dapo
