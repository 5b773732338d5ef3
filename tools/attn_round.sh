# BERT loop: tcgen05 attention parity + timing vs the mma.sync path
timeout 300 python -m pytest tests/test_gpu_engine.py tests/test_gpu_headline.py -q -x -k bert --timeout 120 -s -p no:cacheprovider 2>&1 | grep -E "bert|passed|failed|Error|error" | tail -12
echo "== tcgen05 attention"; timeout 200 python tools/profile_family.py --family bert --batches 8,64,256 | cut -c1-110
echo "== mma.sync attention"; SSN_TC_DEBUG=8388608 timeout 200 python tools/profile_family.py --family bert --batches 8,64,256 | cut -c1-110
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:attention --csv --log-file gpurun_out/attn_metrics.csv python tools/prof_forward.py --family bert --batch 64 --steps 1 --warmup 0 --subnets max > /dev/null 2>&1
python tools/dw_table.py gpurun_out/attn_metrics.csv | tail -4
