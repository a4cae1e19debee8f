# GRPO step rate for a few instantiated scan pipeline shapes (SRT_SCAN_ROWS) in the bench
O=gpurun_out/sv; mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for v in "8,10,4,4,32,1,2,0" "8,10,4,4,32,1,2,1" "8,11,4,4,32,1,2,0" "8,12,4,4,32,1,2,0" "8,10,4,4,32,0,2,0"; do
  SRT_SCAN_ROWS=$v $B > $O/v_$v.log 2>&1
  echo "$v $(tail -1 $O/v_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done
