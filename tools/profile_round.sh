# One profiling pass for profiles/ (run under gpurun): bench line, ncu launch
# list, ncu --set full captures of the scan and of the tree kernels.
# Usage: bash tools/profile_round.sh <tag>
set -x
T=${1:-v6}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_$T.log 2>&1
BENCH_ROWS_LOG=1 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 2 --warmup 4 > gpurun_out/rows_$T.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/launch_bench_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_scan_rows" -s 3 -c 1 -o gpurun_out/scan_$T python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > gpurun_out/ncu_scan_$T.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_draft|k_insert_cursor|k_accept" -s 9 -c 3 -o gpurun_out/tree_$T python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > gpurun_out/ncu_tree_$T.log 2>&1
grep "warm-up step" gpurun_out/rows_$T.log
ls -la gpurun_out
