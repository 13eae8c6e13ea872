mkdir -p gpurun_out/fuse
timeout 900 python -m pytest tests/test_gpu_parity_benched.py tests/test_gpu_parity.py -m gpu -x -q -k "cfg3 or RMC or forward_many or merged or queue or edges" 2>&1 | tail -3
timeout 600 python tools/env_sweep.py --workload cfg3-rmc2 --depth 16 --reps 3 "RS_FUSE_INTER=0" "RS_FUSE_INTER=1" 2>&1 | tail -1
timeout 600 python tools/env_sweep.py --workload rmc1 --depth 16 --reps 3 "RS_FUSE_INTER=0" "RS_FUSE_INTER=1" 2>&1 | tail -1
timeout 600 python tools/env_sweep.py --workload cfg3-rmc3 --depth 16 --reps 3 "RS_FUSE_INTER=0" "RS_FUSE_INTER=1" 2>&1 | tail -1
