# The fused tree step beside the scan: parity vs the step after the scan, then
# step rates for several SM splits (run under gpurun).  Usage: bash tools/probe_overlap.sh <tag>
T=${1:-o1}
O=gpurun_out/$T
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_bench.py -m gpu -x -q -k "beside_scan" > $O/pytest_overlap.log 2>&1; tail -3 $O/pytest_overlap.log
B="timeout 240 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 1024 --steps 20 --warmup 4"
$B --step-overlap 16 --graph 0 > $O/bench_ov16_eager.log 2>&1
for g in 0 8 16 24; do $B --step-overlap $g > $O/bench_ov$g.log 2>&1; done
ls -la $O
