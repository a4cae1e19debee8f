# development sweep of the scan pipeline shapes (SRT_SCAN_ROWS), rl-mix and peaked rows
set -x
mkdir -p gpurun_out
for c in ${SWEEP:-"4,12,4,4,32,0" "4,12,4,4,32,1" "4,12,5,3,32,1" "4,16,4,4,32,1" "6,12,4,4,32,1" "8,12,4,4,32,1" "4,8,4,4,32,1"}; do
  echo "== $c" >> gpurun_out/scan_sweep.txt
  SRT_SCAN_DEBUG=8 SRT_SCAN_ROWS=$c timeout 120 python tools/scan_probe.py --rows 20000 --profiles rl-mix,peaked,moderate --iters 6 >> gpurun_out/scan_sweep.txt 2>&1
done
