mkdir -p gpurun_out/gru2g
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gru_tc -s 1 -c 1 -o gpurun_out/gru2g/gru2g python tools/run_once.py --model DIEN --L 100 --S 300 --fc tf32 --reps 3 > gpurun_out/gru2g/ncu.log 2>&1
RS_GRU_2G=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gru_tc -s 1 -c 1 -o gpurun_out/gru2g/gru1g python tools/run_once.py --model DIEN --L 100 --S 300 --fc tf32 --reps 3 >> gpurun_out/gru2g/ncu.log 2>&1
tail -3 gpurun_out/gru2g/ncu.log
