# microbench conv cases (warm L2 ncu device time) under several env settings:
#   bash tools/ab_mb_env.sh "4,5,7" "SSN_TC_KPS2_NK=0" "SSN_TC_KPS2_NK=8 SSN_TC_DEBUG=12" ...
C=$1; shift
mkdir -p gpurun_out/abmb
i=0
for v in "$@"; do
  env $v CASES=$C timeout 300 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
    --log-file gpurun_out/abmb/e$i.csv python tools/microbench_conv.py > /dev/null 2>&1
  python - "$i" "$v" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/abmb/e{sys.argv[1]}.csv")) if len(r) > 10]
ix = {h: i for i, h in enumerate(rows[0])}
seq = [float(r[ix["Metric Value"]].replace(",", "")) / 1e3 for r in rows[1:]
       if r[ix["Metric Name"]] == "gpu__time_duration.sum" and "conv_" in r[ix["Kernel Name"]]]
print(f"{sys.argv[2]:40s}", " ".join(f"{sorted(seq[b:b + 13])[6]:7.1f}" for b in range(0, len(seq), 13)))
PY
  i=$((i+1))
done
