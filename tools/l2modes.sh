# scan L2 policy modes in the GRPO / PPO step (SRT_SCAN_ROWS hint field)
O=gpurun_out/l2m; mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for h in 0 1 2 3 4; do for cfgn in grpo ppo; do
  SRT_SCAN_ROWS=8,10,4,4,32,$h,2,0 $B --config $cfgn > $O/${cfgn}_h$h.log 2>&1
  echo "$cfgn h$h $(tail -1 $O/${cfgn}_h$h.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done; done
