# per-launch depthwise table (ncu device time, DRAM bytes, GB/s, SM %, FMA %) of one
# OFA-MBv3 bs256 forward per subnet: bash tools/dwprof.sh [min max]
mkdir -p gpurun_out/dw
for s in ${@:-min max}; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none -k regex:dw --csv --log-file gpurun_out/dw/dw_$s.csv python tools/prof_forward.py --family mbv3 --batch 256 --steps 1 --warmup 0 --subnets $s > /dev/null 2>&1
  python tools/dw_table.py gpurun_out/dw/dw_$s.csv > gpurun_out/dw/dw_ncu_mbv3_${s}_bs256.txt
done
