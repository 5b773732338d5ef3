# warm-L2 (ncu --cache-control none) per-launch device times of one bench sweep
# forward per subnet, attributed to plan ops (tools/attribute.py)
mkdir -p gpurun_out/warm
cd /root/repo
B=${B:-64}
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/warm/launches_b$B.csv python tools/prof_forward.py --batch $B --warmup 1 --steps 1 > gpurun_out/warm/pf_b$B.log 2>&1
python tools/attribute.py gpurun_out/warm/launches_b$B.csv --batch $B --top 200 --json gpurun_out/warm/attr_b$B.json > gpurun_out/warm/attr_b$B.txt 2>&1
