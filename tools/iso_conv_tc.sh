# conv_tc isolation (SSN_TC_DEBUG modes) on microbench cases, warm L2 (ncu --cache-control none)
# usage: ISO_CASES=6,7 ISO_DBG="0 2 4 8" bash tools/iso_conv_tc.sh ; results in gpurun_out/iso/
mkdir -p gpurun_out/iso
for d in ${ISO_DBG:-0 1 2 4 8 12 14}; do
  SSN_TC_DEBUG=$d CASES=${ISO_CASES:-4,5,7,30,31,32} timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/iso/mb_$d.csv python tools/microbench_conv.py > gpurun_out/iso/mb_$d.log 2>&1
done
python - <<'PY'
import csv, glob, os
res = {}
for f in sorted(glob.glob("gpurun_out/iso/mb_*.csv")):
    d = os.path.basename(f)[3:-4]
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    ix = {h: i for i, h in enumerate(rows[0])}
    seq = [float(r[ix["Metric Value"]].replace(",", "")) / 1e3 for r in rows[1:]
           if r[ix["Metric Name"]] == "gpu__time_duration.sum" and "conv_" in r[ix["Kernel Name"]]]
    res[d] = [sorted(seq[b:b + 13])[6] for b in range(0, len(seq), 13)]
cases = sorted(int(c) for c in os.environ.get("ISO_CASES", "4,5,7,30,31,32").split(","))
print("case " + " ".join(f"{'d' + d:>9}" for d in res))
for i, c in enumerate(cases):
    print(f"{c:4d} " + " ".join(f"{res[d][i]:9.1f}" if i < len(res[d]) else "        -" for d in res))
PY
