# DAPO: the fused tree step vs the separate kernels after the ranked hub rebuilds
O=gpurun_out/df; mkdir -p $O
B="timeout 400 python bench.py --config dapo --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for rep in 1 2; do
  $B --fused-step 1 > $O/fused_$rep.log 2>&1
  $B --fused-step 0 > $O/sep_$rep.log 2>&1
done
for f in $O/*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
