# depthwise loop: op parity, MBv3 engine parity, family timing, dw ncu table
timeout 300 python -m pytest tests/test_gpu_ops.py -q -x -k dw > gpurun_out/dw_tests.log 2>&1; tail -3 gpurun_out/dw_tests.log
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_headline.py -q -x -k mbv3 -s > gpurun_out/mbv3_tests.log 2>&1; grep -E "mbv3|passed|failed|Error" gpurun_out/mbv3_tests.log | tail -12
timeout 300 python tools/profile_family.py --family mbv3 --batches 16,64,256 > gpurun_out/mbv3_family.log 2>&1; tail -12 gpurun_out/mbv3_family.log
for S in min max; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size --clock-control none -k regex:dw --csv --log-file gpurun_out/dw_metrics_$S.csv python tools/prof_forward.py --family mbv3 --batch 256 --steps 1 --warmup 0 --subnets $S > /dev/null 2>&1
python tools/dw_table.py gpurun_out/dw_metrics_$S.csv
done
