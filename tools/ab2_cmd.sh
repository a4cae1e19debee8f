timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_path_verify.py -m gpu -x -q > gpurun_out/ab2_pytest.log 2>&1; tail -2 gpurun_out/ab2_pytest.log
bash tools/probe_ab.sh ab2 base grpo ppo
timeout 300 python tools/scan_probe.py --rows 18944 --profiles rl-mix,peaked --iters 6 > gpurun_out/ab2/probe_A.txt 2>&1
SRT_LIB=abtest/libsrt_base.so timeout 300 python tools/scan_probe.py --rows 18944 --profiles rl-mix,peaked --iters 6 > gpurun_out/ab2/probe_B.txt 2>&1
