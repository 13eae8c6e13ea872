timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for w in cfg3-rmc2 cfg1-rmc1 rmc2; do
  timeout 300 python tools/env_sweep.py --workload $w --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_SLS_WAVES=2" 2>&1 | tail -1 | sed "s/^/$w /"
done
for w in cfg5-din din; do
  timeout 300 python tools/env_sweep.py --workload $w --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_DIN_WAVES=4" "RS_DIN_WAVES=2" "RS_DIN_WAVES=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
for w in ncf wnd mt-wnd; do
  timeout 300 python tools/env_sweep.py --workload $w --depth 16 --reps 3 --n 1024 "RS_X=default" "RS_CONCAT_WAVES=2" "RS_CONCAT_WAVES=1" 2>&1 | tail -1 | sed "s/^/$w /"
done
timeout 900 python tools/sls_iso.py --sizes 322,1000 "RS_X=default" 2>&1 | tail -1
