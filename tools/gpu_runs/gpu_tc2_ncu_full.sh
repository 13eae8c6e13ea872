mkdir -p gpurun_out/tc2ncu
RS_TC2=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fc_tc2 -s 3 -c 1 -o gpurun_out/tc2ncu/tc2_mtwnd1024 python tools/run_once.py --workload mt-wnd --S 1024 --fc tf32 --reps 2 > gpurun_out/tc2ncu/log.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fc_tc_kernel -s 3 -c 1 -o gpurun_out/tc2ncu/tc1_mtwnd1024 python tools/run_once.py --workload mt-wnd --S 1024 --fc tf32 --reps 2 >> gpurun_out/tc2ncu/log.txt 2>&1
tail -2 gpurun_out/tc2ncu/log.txt
