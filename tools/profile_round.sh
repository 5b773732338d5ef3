# Round profiling bundle (1 GPU): bench lines, launch lists, ncu --set full
# metrics of the tcgen05 conv kernels.  Outputs under gpurun_out/round/.
set -u
O=${O:-gpurun_out/round}
mkdir -p $O
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_r50_bs64.csv \
  python tools/prof_forward.py --steps 1 --warmup 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_mbv3_bs256.csv \
  python tools/prof_forward.py --family mbv3 --batch 256 --steps 1 --warmup 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bert_bs64.csv \
  python tools/prof_forward.py --family bert --batch 64 --steps 1 --warmup 1 > /dev/null 2>&1
# full sections for every conv launch of one max-subnet forward (bs64)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:conv_ --csv --log-file $O/ncu_conv_sweep_bs64.csv \
  python tools/prof_forward.py --steps 1 --warmup 0 > /dev/null 2>&1
python tools/ncu_table.py $O/ncu_conv_sweep_bs64.csv > $O/ncu_conv_sweep_bs64.md

ls -la $O
# one --set full capture of three conv_tc launches of the max subnet (stage-3 3x3 + 1x1s)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conv_tc -s 30 -c 3 \
  -o /tmp/conv_full python tools/prof_forward.py --steps 1 --warmup 0 --subnets max > /dev/null 2>&1
ncu -i /tmp/conv_full.ncu-rep --page details --csv > $O/ncu_full_conv_tc_max.csv 2>/dev/null
ls -la $O
# summaries (text) next to the raw captures
python tools/launches.py $O/launches_r50_bs64.csv > $O/launches_r50_bs64_summary.txt 2>&1
python tools/launches.py $O/launches_mbv3_bs256.csv > $O/launches_mbv3_bs256_summary.txt 2>&1
python tools/launches.py $O/launches_bert_bs64.csv > $O/launches_bert_bs64_summary.txt 2>&1
python tools/attribute.py $O/launches_r50_bs64.csv --top 60 > $O/attributed_r50_bs64.txt 2>&1
