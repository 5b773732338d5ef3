# conv_tc isolation (SSN_TC_DEBUG modes) on the 1x1 microbench cases, warm L2 (ncu --cache-control none)
set -x; mkdir -p gpurun_out/iso
cd /root/repo
for d in 0 1 2 4 8 12 14; do
  SSN_TC_DEBUG=$d CASES=32,30,7,31,4,5,39,40 timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/iso/mb_$d.csv python tools/microbench_conv.py > gpurun_out/iso/mb_$d.log 2>&1
done
SSN_TC_DEBUG=32 CASES=32,30,7 timeout 120 python tools/microbench_conv.py > gpurun_out/iso/prof32.log 2>&1
