for k in 0 1 2 3 4 7; do echo "== skip $k"; SRT_INS_SKIP=$k timeout 200 python tools/insert_probe.py 2>&1 | grep "alone"; done
