# R50 sweep launch list + per-conv-launch DRAM / tensor-pipe table, attributed to plan ops
O=gpurun_out/r50prof; mkdir -p $O
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_forward.py --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py $O/launches.csv > $O/launches_summary.txt 2>&1; head -20 $O/launches_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:conv_ --csv --log-file $O/ncu_conv.csv python tools/prof_forward.py --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_table.py $O/ncu_conv.csv > $O/ncu_conv.md 2>&1; tail -3 $O/ncu_conv.md

