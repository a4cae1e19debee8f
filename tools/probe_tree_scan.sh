# Diagnostic pass (run under gpurun): where the tree step's slowest prompt and
# the scan's per-launch fixed cost go, and how the scan / the tree step behave
# on a subset of the SMs.  Usage: bash tools/probe_tree_scan.sh <tag>
T=${1:-p1}
O=gpurun_out/$T
mkdir -p $O
B="timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 10 --warmup 3"
for g in 118 128 138; do SRT_SCAN_GRID=$g $B > $O/bench_scangrid_$g.log 2>&1; done
for g in 10 20 30 40; do SRT_TREE_GRID=$g $B > $O/bench_treegrid_$g.log 2>&1; done
SRT_STEP_PROF=1 $B > $O/step_prof_grpo.log 2>&1
SRT_STEP_PROF=1 $B --config ppo > $O/step_prof_ppo.log 2>&1
for r in 1184 4736 18944 33792; do
  timeout 300 python tools/scan_probe.py --rows $r --profiles rl-mix,peaked --iters 6 > $O/scan_rows_$r.txt 2>&1
done
timeout 600 python tools/insert_probe.py --config grpo > $O/insert_probe_grpo.txt 2>&1
ls -la $O
