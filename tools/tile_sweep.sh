# Per-op device time of the R50 sweep under forced tile configurations
# (ncu launch lists -> tools/attribute.py JSON), for tuning choose_bn / pairs.
#   bash tools/tile_sweep.sh   -> gpurun_out/tile_<i>.json, one per config
i=0
CFGS=${CFGS:-"X=0 SSN_TC_FORCE_BN=256 SSN_TC_FORCE_BN=128 SSN_TC_PAIR_MIN_NK=1"}
for cfg in $CFGS; do
  env $cfg timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/tile_$i.csv python tools/prof_forward.py --steps 1 --warmup 1 > /dev/null 2>&1
  python tools/attribute.py /tmp/tile_$i.csv --top 0 --json gpurun_out/tile_$i.json > /tmp/tile_$i.txt
  head -4 /tmp/tile_$i.txt
  echo "cfg $i: $cfg"
  i=$((i + 1))
done
