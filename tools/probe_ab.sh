# A/B step rates: the working-tree library vs abtest/libsrt_<B>.so (run under
# gpurun).  Usage: bash tools/probe_ab.sh <tag> <B> [configs...]
T=$1; BL=$2; shift 2
O=gpurun_out/$T
mkdir -p $O
B="timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 --parity-rows 0 --steps 30 --warmup 4"
for cfgn in ${@:-grpo}; do
  for rep in 1 2; do
    $B --config $cfgn > $O/${cfgn}_A$rep.log 2>&1
    SRT_LIB=abtest/libsrt_$BL.so $B --config $cfgn > $O/${cfgn}_B$rep.log 2>&1
  done
done
for f in $O/*.log; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['mean_us'],1) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"; done
