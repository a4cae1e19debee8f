# L2 policy of the scan's TMA loads: evict_first (default) vs none, every config
O=gpurun_out/l2; mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for cfgn in grpo ppo dapo; do for rep in 1 2; do
  $B --config $cfgn > $O/${cfgn}_first_$rep.log 2>&1
  SRT_SCAN_ROWS=8,10,4,4,32,0,2,0 $B --config $cfgn > $O/${cfgn}_none_$rep.log 2>&1
done; done
$B --dtype f32 > $O/f32_first.log 2>&1
SRT_SCAN_ROWS=8,10,4,4,32,0,2,0 $B --dtype f32 > $O/f32_none.log 2>&1
for f in $O/*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
timeout 300 python tools/scan_probe.py --rows 18944 --profiles rl-mix,peaked --iters 6 2>&1 | grep scan
SRT_SCAN_ROWS=8,10,4,4,32,0,2,0 timeout 300 python tools/scan_probe.py --rows 18944 --profiles rl-mix,peaked --iters 6 2>&1 | grep scan
