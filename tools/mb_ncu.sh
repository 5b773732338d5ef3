# per-kernel device time (ncu gpu__time_duration) of the conv microbench cases,
# optionally under SSN_TC_DEBUG isolation modes: bash tools/mb_ncu.sh "0 7" "0,1,11"
for d in $1; do
  SSN_TC_DEBUG=$d CASES=$2 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/mb_$d.csv python tools/microbench_conv.py > /dev/null 2>&1
  python - "$d" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"/tmp/mb_{sys.argv[1]}.csv")) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
seq = [(r[ix["Kernel Name"]].split("(")[0].split("<")[0][-20:], float(r[ix["Metric Value"]].replace(",", "")) / 1e3) for r in rows[1:] if r[ix["Metric Name"]] == "gpu__time_duration.sum" and "conv_" in r[ix["Kernel Name"]]]
# 13 launches per case (3 warm-up + 10 timed): report the median of each block of 13
for b in range(0, len(seq), 13):
    blk = sorted(v for _, v in seq[b:b + 13])
    print(f"dbg={sys.argv[1]} case#{b // 13} {seq[b][0]:>20} {blk[len(blk) // 2]:8.1f} us")
PY
done
