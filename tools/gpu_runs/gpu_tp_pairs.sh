mkdir -p gpurun_out
TP_CASES="mt-wnd:256,mt-wnd:1024,wnd:1024" TP_TAG=_one timeout 900 python tools/tensor_profile.py > gpurun_out/tp_one.json 2> gpurun_out/tp_one.err
RS_TC2=2 TP_CASES="mt-wnd:256,mt-wnd:1024,wnd:1024" TP_TAG=_pair timeout 900 python tools/tensor_profile.py > gpurun_out/tp_pair.json 2> gpurun_out/tp_pair.err
tail -3 gpurun_out/tp_one.err gpurun_out/tp_pair.err
