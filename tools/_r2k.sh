timeout 900 python -m pytest tests -m gpu -q -x -k "mbv3 or se" 2>&1 | tail -3
echo "== mbv3"; timeout 300 python tools/profile_family.py --family mbv3 --batches 64,256 | cut -c1-110
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k_mbv3.csv python tools/prof_forward.py --family mbv3 --batch 256 --steps 1 --warmup 1 --subnets max > /dev/null 2>&1
python tools/launches.py gpurun_out/r2k_mbv3.csv 2>/dev/null | head -14
