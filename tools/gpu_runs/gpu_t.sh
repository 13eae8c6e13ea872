#!/bin/bash
mkdir -p gpurun_out
for SK in 0 7 2; do
  timeout 900 ncu --replay-mode app-range --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum python tools/range_traffic.py --n 256 --skip $SK > gpurun_out/range_$SK.csv 2> gpurun_out/range_$SK.err
done
