timeout 400 python tools/env_sweep.py --workload ncf --depth 16 --reps 3 "RS_X=default" "RS_TC2_ALL=1" 2>&1 | tail -1 | sed "s/^/ncf /"
timeout 400 python -m pytest tests/test_gpu_parity_benched.py -m gpu -q -k "WND or cta_pair" 2>&1 | tail -1
