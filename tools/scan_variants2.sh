# scan pipeline shapes without the L2 policy (the r02 v6 default) in the GRPO / PPO step
O=gpurun_out/sv2; mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for v in "8,10,4,4,32,0,2,0" "8,11,4,4,32,0,2,0" "8,10,6,3,32,0,2,0" "12,9,6,3,32,0,3,0" "8,10,4,4,32,0,2,1"; do for cfgn in grpo ppo; do
  SRT_SCAN_ROWS=$v $B --config $cfgn > $O/${cfgn}_$v.log 2>&1
  echo "$cfgn $v $(tail -1 $O/${cfgn}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done; done
