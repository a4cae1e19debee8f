# final state check: GPU suite, smoke, default bench line
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; tail -1 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -1 gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_grpo.log 2>&1; tail -1 gpurun_out/final/bench_grpo.log | cut -c1-300
