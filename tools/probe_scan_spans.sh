# Per-CTA spans of the scan inside the GRPO / PPO step (a -DSRT_SCAN_PROF build,
# tools/build_ab.sh prof HEAD with NVFLAGS=-DSRT_SCAN_PROF).  Usage: bash tools/probe_scan_spans.sh <tag>
T=${1:-s1}
O=gpurun_out/$T
mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 3 --warmup 3 --graph 0"
SRT_LIB=abtest/libsrt_prof.so SRT_SCAN_DEBUG=128 $B > $O/spans_grpo.log 2>&1
SRT_LIB=abtest/libsrt_prof.so SRT_SCAN_DEBUG=128 $B --config ppo > $O/spans_ppo.log 2>&1
SRT_LIB=abtest/libsrt_prof.so SRT_SCAN_DEBUG=192 $B > $O/waits_grpo.log 2>&1
ls -la $O
