set -x
mkdir -p gpurun_out
BENCH_ROWS_LOG=1 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 2 --warmup 4 > gpurun_out/rows.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v4.csv python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 > gpurun_out/launch_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_scan_rows" -s 3 -c 1 -o gpurun_out/scan_v4 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > gpurun_out/ncu_scan.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_draft|k_insert_cursor|k_accept" -s 9 -c 3 -o gpurun_out/tree_v4 python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > gpurun_out/ncu_tree.log 2>&1
grep "warm-up step" gpurun_out/rows.log
ls -la gpurun_out
