# warm-L2 (ncu --cache-control none) per-launch device times of one bench sweep
# forward per subnet, attributed to plan ops (tools/attribute.py); TAG names the run
mkdir -p gpurun_out/warm
B=${B:-64}; TAG=${TAG:-b$B}
timeout 600 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/warm/launches_$TAG.csv python tools/prof_forward.py --batch $B --warmup 1 --steps 1 > gpurun_out/warm/pf_$TAG.log 2>&1
python tools/attribute.py gpurun_out/warm/launches_$TAG.csv --batch $B --top 200 --json gpurun_out/warm/attr_$TAG.json > gpurun_out/warm/attr_$TAG.txt 2>&1
