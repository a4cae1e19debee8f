# Round-2 measurement pass (run under gpurun): bench lines for every config /
# dtype / profile / verify mode, the full-draft scan stress probe, the ncu
# launch list and ncu --set full captures of the scan, tree and LM-head
# kernels.
# Usage: bash tools/profile_r02.sh <tag>
T=${1:-v1}
O=gpurun_out/$T
mkdir -p $O
B="timeout 600 python bench.py"
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
$B > $O/bench_grpo.log 2>&1
$B --fused-step 0 --no-cpu-baseline --e2e-steps 0 > $O/bench_grpo_unfused_step.log 2>&1
$B --dtype f32 --no-cpu-baseline > $O/bench_grpo_f32.log 2>&1
for p in peaked moderate flat; do $B --profile $p --no-cpu-baseline --e2e-steps 0 > $O/bench_grpo_$p.log 2>&1; done
$B --config ppo --no-cpu-baseline > $O/bench_ppo.log 2>&1
$B --config dapo --no-cpu-baseline > $O/bench_dapo.log 2>&1
$B --verify lmhead --no-cpu-baseline > $O/bench_grpo_lmhead.log 2>&1
$B --verify path --no-cpu-baseline > $O/bench_grpo_path.log 2>&1
$B --config b200x8 --sharded --no-cpu-baseline --steps 10 --e2e-steps 0 > $O/bench_b200x8_rank.log 2>&1
timeout 300 python tools/scan_probe.py --rows 33792 --profiles rl-mix,peaked,moderate,flat --iters 6 > $O/scan_fulldraft.txt 2>&1
timeout 300 python tools/scan_probe.py --rows 16896 --profiles rl-mix,peaked,flat --iters 6 --dtype f32 > $O/scan_fulldraft_f32.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --no-cpu-baseline --e2e-steps 0 --steps 3 --warmup 3 > $O/launch_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_scan_rows" -s 3 -c 1 -o $O/scan python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > $O/ncu_scan.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tree_step" -s 3 -c 1 -o $O/tree python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > $O/ncu_tree.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_draft|k_accept|k_hub_refresh" -s 12 -c 3 -o $O/tree_unfused python bench.py --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 --fused-step 0 > $O/ncu_tree_unfused.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_lmhead_sample" -s 3 -c 1 -o $O/lmhead python bench.py --verify lmhead --no-cpu-baseline --e2e-steps 0 --steps 1 --warmup 4 > $O/ncu_lmhead.log 2>&1
# (compute-sanitizer is closed on this pool since r02 v3: no sanitizer legs)
ls -la $O
