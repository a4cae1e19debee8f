# scan default (8 stream, 11 tail warps): scan parity, then A/B vs (8, 10) via SRT_SCAN_ROWS
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_path_verify.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ab7_pytest.log 2>&1; tail -2 gpurun_out/ab7_pytest.log
O=gpurun_out/ab7; mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for cfgn in grpo ppo dapo; do for rep in 1 2; do
  $B --config $cfgn > $O/${cfgn}_A$rep.log 2>&1
  SRT_SCAN_ROWS=8,10,4,4,32,0,2,0 $B --config $cfgn > $O/${cfgn}_B$rep.log 2>&1
done; done
$B --dtype f32 > $O/f32_A.log 2>&1
SRT_SCAN_ROWS=8,10,4,4,32,0,2,0 $B --dtype f32 > $O/f32_B.log 2>&1
for f in $O/*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
