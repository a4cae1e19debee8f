timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; tail -2 gpurun_out/pt_all.log
timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_nocpu.log 2>&1
timeout 400 python bench.py --config dapo --no-cpu-baseline --e2e-steps 0 --steps 20 > gpurun_out/bench_dapo.log 2>&1
timeout 300 python bench.py --config ppo --no-cpu-baseline --e2e-steps 0 --steps 20 > gpurun_out/bench_ppo.log 2>&1
